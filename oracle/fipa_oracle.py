"""ORACLE / TEST INFRASTRUCTURE ONLY -- never imported by the product.

A float64 numpy restatement of the reference FlashIPA layer
(/root/reference/proj, CPU C++20).  Every function cites the reference
file:line it restates.  It is pinned against the reference itself: the
compiled reference (oracle/_ref/libfipa_ref.so, built by oracle/Makefile from
the reference's own sources) produced the committed fixtures under
tests/golden/ (script: oracle/gen_golden.py), and tests/test_oracle.py checks
this restatement against them.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
# ln(e - 1): raw gamma whose softplus is exactly 1 (proj/src/ipa.cpp:30).
GAMMA_RAW_UNIT = 0.5413248546129181


# --------------------------------------------------------------------------- rng
def _mix64_vec(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer, vectorised (proj/src/rng.cpp:11-16)."""
    z = z.astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class Rng:
    """Counter-based generator (proj/include/fipa/rng.hpp:11-30, proj/src/rng.cpp:18-41).

    Draw n = mix64(seed + n*golden); uniform on (0,1] = ((u >> 11) + 1) * 2^-53;
    Box-Muller with the sine variate cached as the next draw.  Transcendentals
    go through `math` (glibc libm, the same one the reference links) so the
    stream is bit-identical to the C++ one.
    """

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self.counter = 0
        self.spare = 0.0
        self.have_spare = False

    def _uniforms(self, n: int) -> np.ndarray:
        idx = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            u = _mix64_vec(np.uint64(self.seed) + idx * np.uint64(GOLDEN))
        return ((u >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0**-53

    def uniform(self) -> float:
        return float(self._uniforms(1)[0])

    def gaussian(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        u1, u2 = self._uniforms(2)
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 2.0 * math.pi * u2
        self.spare = radius * math.sin(angle)
        self.have_spare = True
        return radius * math.cos(angle)

    def gaussians(self, n: int) -> np.ndarray:
        """n consecutive gaussian() draws (bit-identical to n scalar calls)."""
        out = np.empty(n, dtype=np.float64)
        pos = 0
        if n and self.have_spare:
            out[0] = self.spare
            self.have_spare = False
            pos = 1
        pairs = (n - pos + 1) // 2
        if pairs:
            u = self._uniforms(2 * pairs)
            u1, u2 = u[0::2], u[1::2]
            log, sqrt, sin, cos, pi2 = math.log, math.sqrt, math.sin, math.cos, 2.0 * math.pi
            vals = np.empty(2 * pairs, dtype=np.float64)
            for p in range(pairs):
                r = sqrt(-2.0 * log(u1[p]))
                a = pi2 * u2[p]
                vals[2 * p] = r * cos(a)
                vals[2 * p + 1] = r * sin(a)
            take = n - pos
            out[pos:] = vals[:take]
            if take < 2 * pairs:
                self.spare = float(vals[-1])
                self.have_spare = True
        return out


def gaussian_tensor(rng: Rng, shape, stddev=1.0, f32=False) -> np.ndarray:
    """proj/src/tensor.cpp:286-290: flat-order draws times stddev, stored at precision."""
    n = int(np.prod(shape))
    vals = stddev * rng.gaussians(n)
    if f32:
        vals = vals.astype(np.float32).astype(np.float64)
    return vals.reshape(shape)


# ------------------------------------------------------------------------ config
@dataclass
class IpaConfig:
    """proj/include/fipa/ipa.hpp:14-32."""

    d_in: int = 32
    d_z: int = 4
    heads: int = 2
    c: int = 8
    n_query: int = 2
    n_value: int = 2
    rank: int = 2
    precision: str = "f64"
    enforce_head_cap: bool = True

    def qk_width(self) -> int:
        return self.c + 5 * self.n_query + self.rank * self.d_z

    def v_width(self) -> int:
        return self.c + 3 * self.n_value + self.rank * self.d_z

    def seg(self) -> int:
        return self.d_z + self.c + 4 * self.n_value

    def validate(self):
        """proj/src/ipa.cpp:12-21."""
        dims = (self.d_in, self.d_z, self.heads, self.c, self.n_query, self.n_value, self.rank)
        if min(dims) <= 0:
            raise ValueError("all IpaConfig dimensions must be positive")
        if self.enforce_head_cap and max(self.qk_width(), self.v_width()) > 256:
            raise ValueError("lifted head width exceeds the cap of 256")

    def as_u64(self):
        return [self.d_in, self.d_z, self.heads, self.c, self.n_query, self.n_value,
                self.rank, 0 if self.precision == "f32" else 1, int(self.enforce_head_cap)]


WEIGHT_NAMES = ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp", "w_bias", "gamma_raw", "w_out", "b_out")


def weight_shapes(cfg: IpaConfig):
    seg = cfg.seg()
    return {
        "w_q": (cfg.d_in, cfg.heads * cfg.c),
        "w_k": (cfg.d_in, cfg.heads * cfg.c),
        "w_v": (cfg.d_in, cfg.heads * cfg.c),
        "w_qp": (cfg.d_in, cfg.heads * cfg.n_query * 3),
        "w_kp": (cfg.d_in, cfg.heads * cfg.n_query * 3),
        "w_vp": (cfg.d_in, cfg.heads * cfg.n_value * 3),
        "w_bias": (cfg.heads, cfg.d_z),
        "gamma_raw": (cfg.heads,),
        "w_out": (cfg.heads * seg, cfg.d_in),
        "b_out": (cfg.d_in,),
    }


def init_weights(cfg: IpaConfig, seed: int) -> dict:
    """IpaWeights::init (proj/src/ipa.cpp:172-193), draw order preserved."""
    cfg.validate()
    rng = Rng(seed)
    f32 = cfg.precision == "f32"
    s_in = 1.0 / math.sqrt(cfg.d_in)
    sh = weight_shapes(cfg)
    w = {}
    for name in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp"):
        w[name] = gaussian_tensor(rng, sh[name], s_in, f32)
    w["w_bias"] = gaussian_tensor(rng, sh["w_bias"], 1.0 / math.sqrt(cfg.d_z), f32)
    g = np.full(sh["gamma_raw"], GAMMA_RAW_UNIT)
    w["gamma_raw"] = g.astype(np.float32).astype(np.float64) if f32 else g
    concat_w = sh["w_out"][0]
    w["w_out"] = gaussian_tensor(rng, sh["w_out"], 1.0 / math.sqrt(concat_w), f32)
    w["b_out"] = np.zeros(sh["b_out"])
    w["w_l"] = math.sqrt(1.0 / 3.0)
    w["w_c"] = math.sqrt(2.0 / (9.0 * cfg.n_query))
    return w


def softplus(x):
    """proj/src/ipa.cpp:25-27 (stable form)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > 0, x + np.log1p(np.exp(-np.abs(x))), np.log1p(np.exp(np.minimum(x, 0))))


# ---------------------------------------------------------------------- geometry
def apply(rot, trans, x):
    """y = R x + t (proj/src/geometry.cpp:63-68); rot [...,3,3], x [...,3]."""
    return np.einsum("...ab,...b->...a", rot, x) + trans


def apply_inverse(rot, trans, x):
    """y = R^T (x - t) (proj/src/geometry.cpp:70-76)."""
    return np.einsum("...ba,...b->...a", rot, x - trans)


def compose(r1, t1, r2, t2):
    """T1 after T2 (proj/src/geometry.cpp:78-90)."""
    return r1 @ r2, np.einsum("...ab,...b->...a", r1, t2) + t1


def random_rototranslation(rng: Rng, translation_scale: float):
    """Normalised Gaussian quaternion -> rotation (proj/src/geometry.cpp:107-132)."""
    while True:
        qw, qx, qy, qz = (rng.gaussian() for _ in range(4))
        qn = math.sqrt(qw * qw + qx * qx + qy * qy + qz * qz)
        if qn >= 1e-12:
            break
    qw, qx, qy, qz = qw / qn, qx / qn, qy / qn, qz / qn
    rot = np.array([
        [1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy)],
        [2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx)],
        [2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)],
    ])
    trans = np.array([translation_scale * rng.gaussian() for _ in range(3)])
    return rot, trans


def random_frames(rng: Rng, L: int, scale: float = 1.0):
    """tests/test_support.hpp:36-44."""
    rots, trans = np.empty((L, 3, 3)), np.empty((L, 3))
    for i in range(L):
        rots[i], trans[i] = random_rototranslation(rng, scale)
    return rots, trans


# -------------------------------------------------------------------- the layer
def _head_major(x, H, w):
    """[L, H*w] -> [H, L, w] (proj/src/ipa.cpp:33-44)."""
    L = x.shape[0]
    return x.reshape(L, H, w).transpose(1, 0, 2)


def project_inputs(s, cfg: IpaConfig, w):
    """proj/src/ipa.cpp:201-217: six bias-free projections, head-major."""
    H, L = cfg.heads, s.shape[0]
    q = _head_major(s @ w["w_q"], H, cfg.c)
    k = _head_major(s @ w["w_k"], H, cfg.c)
    v = _head_major(s @ w["w_v"], H, cfg.c)
    qp = _head_major(s @ w["w_qp"], H, cfg.n_query * 3).reshape(H, L, cfg.n_query, 3)
    kp = _head_major(s @ w["w_kp"], H, cfg.n_query * 3).reshape(H, L, cfg.n_query, 3)
    vp = _head_major(s @ w["w_vp"], H, cfg.n_value * 3).reshape(H, L, cfg.n_value, 3)
    return q, k, v, qp, kp, vp


def bias_factors(z1, z2, per_head_w):
    """proj/src/pair_features.cpp:141-163: b1[i,h]=flat z1[i]; b2[j,h]=flat(w_h (.) z2[j])."""
    L, r, dz = z1.shape
    H = per_head_w.shape[0]
    b1 = np.broadcast_to(z1.reshape(L, 1, r * dz), (L, H, r * dz)).copy()
    b2 = (per_head_w[None, :, None, :] * z2[:, None, :, :]).reshape(L, H, r * dz)
    return b1, b2


def lift_qkv(s, z1, z2, rot, trans, cfg: IpaConfig, w):
    """Lifted rows exactly as flash_ipa_forward builds them.

    w_l fold: proj/src/flash_ipa.cpp:161-167; lifts: flash_ipa.cpp:23-126.
    Returns q_hat, k_hat [H, L, qk_width] and v_hat [H, L, v_width].
    """
    H, L, Nq, Nv = cfg.heads, s.shape[0], cfg.n_query, cfg.n_value
    q, k, v, qp, kp, vp = project_inputs(s, cfg, w)
    b1, b2 = bias_factors(z1, z2, w["w_l"] * w["w_bias"])
    gamma = softplus(w["gamma_raw"])
    gq = apply(rot[None, :, None], trans[None, :, None], qp)  # [H, L, Nq, 3]
    gk = apply(rot[None, :, None], trans[None, :, None], kp)
    gv = apply(rot[None, :, None], trans[None, :, None], vp)
    g = (gamma * w["w_l"] * w["w_c"])[:, None, None]  # [H,1,1]
    q_hat = np.concatenate([
        q, gq.reshape(H, L, 3 * Nq), (gq ** 2).sum(-1), np.ones((H, L, Nq)),
        b1.transpose(1, 0, 2)], axis=-1)
    k_hat = np.concatenate([
        w["w_l"] / math.sqrt(cfg.c) * k, g * gk.reshape(H, L, 3 * Nq),
        np.broadcast_to(-0.5 * g, (H, L, Nq)), -0.5 * g * (gk ** 2).sum(-1),
        b2.transpose(1, 0, 2)], axis=-1)
    v_hat = np.concatenate([
        v, gv.reshape(H, L, 3 * Nv),
        np.broadcast_to(z2.reshape(1, L, -1), (H, L, cfg.rank * cfg.d_z))], axis=-1)
    return q_hat, k_hat, v_hat


def flash_attention(q, k, v, mask=None):
    """Online-softmax attention, proj/src/attention_kernel.cpp:112-188 / 213-243.

    Restated densely (mathematically identical): key-only mask, no internal
    scale, rows with no valid key come back as zeros (attention_kernel.cpp:184-186).
    q,k [H,L,d], v [H,L,dv].
    """
    s = np.einsum("hid,hjd->hij", q, k)
    if mask is not None:
        s = np.where(np.asarray(mask, bool)[None, None, :], s, -np.inf)
    m = s.max(-1, keepdims=True)
    valid = np.isfinite(m)
    p = np.exp(np.where(valid, s - np.where(valid, m, 0.0), -np.inf))
    l = p.sum(-1, keepdims=True)
    out = np.einsum("hij,hjd->hid", p, v) / np.where(l > 0, l, 1.0)
    return np.where(l > 0, out, 0.0)


def attention_lse(q, k, mask=None):
    """Natural-log LSE per query row (used by backward parity)."""
    s = np.einsum("hid,hjd->hij", q, k)
    if mask is not None:
        s = np.where(np.asarray(mask, bool)[None, None, :], s, -np.inf)
    m = s.max(-1, keepdims=True)
    return (m + np.log(np.exp(s - m).sum(-1, keepdims=True)))[..., 0]


def epilogue_features(o_hat, z1, rot, trans, cfg: IpaConfig):
    """Split / pair-contract / inverse-frame / norms (proj/src/flash_ipa.cpp:171-210).

    o_hat [H, L, v_width] -> feat [L, H*seg], per-head block
    [pair d_z | scalar c | local points 3Nv | norms Nv].
    """
    H, L = o_hat.shape[0], o_hat.shape[1]
    c, Nv, r, dz = cfg.c, cfg.n_value, cfg.rank, cfg.d_z
    pair = o_hat[:, :, c + 3 * Nv:].reshape(H, L, r, dz)
    pair_c = (z1[None] * pair).sum(2)  # [H, L, dz]
    scal = o_hat[:, :, :c]
    gpts = o_hat[:, :, c:c + 3 * Nv].reshape(H, L, Nv, 3)
    loc = apply_inverse(rot[None, :, None], trans[None, :, None], gpts)
    nrm = np.sqrt((loc ** 2).sum(-1))
    blk = np.concatenate([pair_c, scal, loc.reshape(H, L, 3 * Nv), nrm], axis=-1)
    return blk.transpose(1, 0, 2).reshape(L, H * cfg.seg())


def flash_ipa_forward(s, z1, z2, rot, trans, mask, cfg: IpaConfig, w, return_intermediates=False):
    """proj/src/flash_ipa.cpp:141-218 restated at float64."""
    L = s.shape[0]
    mask = np.ones(L, bool) if mask is None else np.asarray(mask, bool)
    if L < 1:
        raise ValueError("empty frame set")
    if not mask.any():  # flash_ipa.cpp:156-159
        out = np.zeros((L, cfg.d_in))
        return (out, {}) if return_intermediates else out
    q_hat, k_hat, v_hat = lift_qkv(s, z1, z2, rot, trans, cfg, w)
    o_hat = flash_attention(q_hat, k_hat, v_hat, mask)
    feat = epilogue_features(o_hat, z1, rot, trans, cfg)
    out = feat @ w["w_out"] + w["b_out"]  # flash_ipa.cpp:212
    out[~mask] = 0.0  # flash_ipa.cpp:213-216
    if return_intermediates:
        return out, dict(q_hat=q_hat, k_hat=k_hat, v_hat=v_hat, o_hat=o_hat, feat=feat)
    return out


def reference_forward(s, z1, z2, rot, trans, mask, cfg: IpaConfig, w):
    """Quadratic restatement of proj/src/ipa.cpp:244-310 (dense z, dense logits)."""
    L = s.shape[0]
    mask = np.ones(L, bool) if mask is None else np.asarray(mask, bool)
    if not mask.any():
        return np.zeros((L, cfg.d_in))
    z = np.einsum("ird,jrd->ijd", z1, z2)  # pair_features.cpp:123-139
    bias = np.einsum("hd,ijd->hij", w["w_bias"], z)  # ipa.cpp:102-119
    q, k, v, qp, kp, vp = project_inputs(s, cfg, w)
    gq = apply(rot[None, :, None], trans[None, :, None], qp)
    gk = apply(rot[None, :, None], trans[None, :, None], kp)
    gv = apply(rot[None, :, None], trans[None, :, None], vp)
    gamma = softplus(w["gamma_raw"])
    dist = ((gq[:, :, None] - gk[:, None, :]) ** 2).sum((-1, -2))
    logits = w["w_l"] * (np.einsum("hic,hjc->hij", q, k) / math.sqrt(cfg.c) + bias
                         - (0.5 * gamma * w["w_c"])[:, None, None] * dist)  # ipa.cpp:95-96
    logits = np.where(mask[None, None, :], logits, -np.inf)
    attn = np.exp(logits - logits.max(-1, keepdims=True))
    attn /= attn.sum(-1, keepdims=True)
    agg_z = np.einsum("hij,ijd->hid", attn, z)
    agg_v = np.einsum("hij,hjc->hic", attn, v)
    agg_p = np.einsum("hij,hjpx->hipx", attn, gv)
    loc = apply_inverse(rot[None, :, None], trans[None, :, None], agg_p)
    nrm = np.sqrt((loc ** 2).sum(-1))
    H = cfg.heads
    blk = np.concatenate([agg_z, agg_v, loc.reshape(H, L, -1), nrm], -1)
    feat = blk.transpose(1, 0, 2).reshape(L, -1)
    out = feat @ w["w_out"] + w["b_out"]
    out[~mask] = 0.0
    return out


def rel_dev(ref, other) -> float:
    """max|a-b| / max|ref| (proj/tests/test_support.hpp:31-34)."""
    ref = np.asarray(ref, np.float64)
    denom = max(float(np.abs(ref).max()) if ref.size else 0.0, np.finfo(np.float64).tiny)
    return float(np.abs(ref - np.asarray(other, np.float64)).max()) / denom


def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float64."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(x))


def round_f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


@dataclass
class Problem:
    s: np.ndarray
    z1: np.ndarray
    z2: np.ndarray
    rot: np.ndarray
    trans: np.ndarray
    mask: np.ndarray = field(default=None)


def make_problem(cfg: IpaConfig, L: int, seed: int, translation_scale: float = 1.0,
                 mask_frac: float = 0.0) -> Problem:
    """Reference-style synthetic inputs (proj/tests/test_support.hpp:36-52):
    s, z1, z2 ~ N(0,1); frames from random_rototranslation(rng, scale)."""
    rng = Rng(seed)
    s = gaussian_tensor(rng, (L, cfg.d_in))
    z1 = gaussian_tensor(rng, (L, cfg.rank, cfg.d_z))
    z2 = gaussian_tensor(rng, (L, cfg.rank, cfg.d_z))
    rot, trans = random_frames(rng, L, translation_scale)
    mask = np.ones(L, bool)
    if mask_frac > 0:
        u = rng._uniforms(L)
        mask = u >= mask_frac
    return Problem(s, z1, z2, rot, trans, mask)


# ---------------------------------------------------------------------- backward
def flash_ipa_backward(s, z1, z2, rot, trans, mask, cfg: IpaConfig, w, dout):
    """Reverse-mode derivative of the layer, float64.

    The reference has no backward (proj/SPEC.md:8, :80); this differentiates the quadratic
    restatement of proj/src/ipa.cpp:244-310 (== flash_ipa_forward, proj/src/flash_ipa.cpp:141-218,
    pinned by tests/test_oracle.py) by hand.  Rotations are treated as free 3x3 matrices, exactly
    as the forward consumes them (geometry.cpp:63-76).  It is pinned against central finite
    differences of the compiled reference forward (tests/test_oracle.py::test_backward_fd).
    Returns a dict with the gradient of sum(out * dout) w.r.t. s, z1, z2, rot, trans and every
    weight tensor (reference names).
    """
    L = s.shape[0]
    H, c, Nq, Nv, r, dz = cfg.heads, cfg.c, cfg.n_query, cfg.n_value, cfg.rank, cfg.d_z
    mask = np.ones(L, bool) if mask is None else np.asarray(mask, bool)
    g = {n: np.zeros_like(np.asarray(w[n], np.float64)) for n in WEIGHT_NAMES}
    g.update(s=np.zeros_like(s), z1=np.zeros_like(z1), z2=np.zeros_like(z2),
             rot=np.zeros_like(rot), trans=np.zeros_like(trans))
    if not mask.any():  # flash_ipa.cpp:156-159: constant zero output
        return g
    wl, wc = w["w_l"], w["w_c"]
    z = np.einsum("ird,jrd->ijd", z1, z2)
    q, k, v, qp, kp, vp = project_inputs(s, cfg, w)
    R, t = rot[None, :, None], trans[None, :, None]
    gq, gk, gv = apply(R, t, qp), apply(R, t, kp), apply(R, t, vp)
    gamma = softplus(w["gamma_raw"])
    diff = gq[:, :, None] - gk[:, None, :]  # [H, i, j, Nq, 3]
    dist = (diff ** 2).sum((-1, -2))
    bias = np.einsum("hd,ijd->hij", w["w_bias"], z)
    logits = wl * (np.einsum("hic,hjc->hij", q, k) / math.sqrt(c) + bias
                   - (0.5 * gamma * wc)[:, None, None] * dist)
    logits = np.where(mask[None, None, :], logits, -np.inf)
    attn = np.exp(logits - logits.max(-1, keepdims=True))
    attn /= attn.sum(-1, keepdims=True)
    agg_z = np.einsum("hij,ijd->hid", attn, z)
    agg_v = np.einsum("hij,hjc->hic", attn, v)
    agg_p = np.einsum("hij,hjpx->hipx", attn, gv)
    y = agg_p - t
    loc = np.einsum("iba,hipb->hipa", rot, y)
    nrm = np.sqrt((loc ** 2).sum(-1))
    blk = np.concatenate([agg_z, agg_v, loc.reshape(H, L, -1), nrm], -1)
    feat = blk.transpose(1, 0, 2).reshape(L, -1)

    dout_m = np.where(mask[:, None], dout, 0.0)  # flash_ipa.cpp:213-216
    g["b_out"] = dout_m.sum(0)
    g["w_out"] = feat.T @ dout_m
    dblk = (dout_m @ w["w_out"].T).reshape(L, H, cfg.seg()).transpose(1, 0, 2)
    d_aggz = dblk[..., :dz]
    d_aggv = dblk[..., dz:dz + c]
    d_loc = dblk[..., dz + c:dz + c + 3 * Nv].reshape(H, L, Nv, 3).copy()
    d_nrm = dblk[..., dz + c + 3 * Nv:]
    safe = np.where(nrm > 0, nrm, 1.0)
    d_loc += np.where(nrm > 0, d_nrm / safe, 0.0)[..., None] * loc
    d_aggp = np.einsum("iab,hipb->hipa", rot, d_loc)
    g["trans"] -= d_aggp.sum((0, 2))
    g["rot"] += np.einsum("hipb,hipa->iba", y, d_loc)

    d_attn = (np.einsum("hid,ijd->hij", d_aggz, z) + np.einsum("hic,hjc->hij", d_aggv, v)
              + np.einsum("hipx,hjpx->hij", d_aggp, gv))
    dzz = np.einsum("hij,hid->ijd", attn, d_aggz)
    dv = np.einsum("hij,hic->hjc", attn, d_aggv)
    dgv = np.einsum("hij,hipx->hjpx", attn, d_aggp)
    dlog = attn * (d_attn - (attn * d_attn).sum(-1, keepdims=True))

    dq = wl / math.sqrt(c) * np.einsum("hij,hjc->hic", dlog, k)
    dk = wl / math.sqrt(c) * np.einsum("hij,hic->hjc", dlog, q)
    dbias = wl * dlog
    g["w_bias"] = np.einsum("hij,ijd->hd", dbias, z)
    dzz += np.einsum("hij,hd->ijd", dbias, w["w_bias"])
    ddist = -0.5 * wl * wc * gamma[:, None, None] * dlog
    dgamma = -0.5 * wl * wc * (dlog * dist).sum((1, 2))
    g["gamma_raw"] = dgamma / (1.0 + np.exp(-np.asarray(w["gamma_raw"], np.float64)))
    dgq = 2.0 * np.einsum("hij,hijpx->hipx", ddist, diff)
    dgk = -2.0 * np.einsum("hij,hijpx->hjpx", ddist, diff)

    g["z1"] = np.einsum("ijd,jrd->ird", dzz, z2)
    g["z2"] = np.einsum("ijd,ird->jrd", dzz, z1)
    dpts = []
    for dgx, x in ((dgq, qp), (dgk, kp), (dgv, vp)):
        g["trans"] += dgx.sum((0, 2))
        g["rot"] += np.einsum("hipa,hipb->iab", dgx, x)
        dpts.append(np.einsum("iab,hipa->hipb", rot, dgx))

    def flat(x):  # [H, L, ...] -> [L, H*...] (inverse of _head_major)
        return x.reshape(H, L, -1).transpose(1, 0, 2).reshape(L, -1)

    for name, dx in (("w_q", dq), ("w_k", dk), ("w_v", dv), ("w_qp", dpts[0]), ("w_kp", dpts[1]),
                     ("w_vp", dpts[2])):
        f = flat(dx)
        g[name] = s.T @ f
        g["s"] += f @ w[name].T
    return g


# ------------------------------------------------------------------------- trunk
# BASELINE cfg3 ("6-layer FrameFlow-style IPA trunk with per-layer backbone frame update").  The
# reference has no trunk, residual or backbone update (proj/SPEC.md:307), so the
# build defines one, FrameFlow-style, from reference pieces: per layer
#   s <- s + flash_ipa_forward(s, z, T)                       (proj/src/flash_ipa.cpp:141-218)
#   u = s . W_bb + b_bb  (Linear(c_s, 6)),  q = (1, u0, u1, u2)/|.|,  dT = (R(q), u[3:6])
#   T <- compose(T, dT) = (R dR, R du + t)                    (proj/src/geometry.cpp:78-90)
# with R(q) the reference's quaternion->matrix map (geometry.cpp:107-132); masked residues keep
# their frames.  Layer l's IPA weights are IpaWeights::init(cfg, Rng(seed + l)); its backbone
# weights are N(0, (0.1/sqrt(d_in))^2) draws from Rng(seed + 1000 + l), bias zero.
def quat_to_rot(qw, qx, qy, qz):
    """Normalised quaternion -> rotation (the matrix of proj/src/geometry.cpp:107-132)."""
    n = np.sqrt(qw * qw + qx * qx + qy * qy + qz * qz)
    qw, qx, qy, qz = qw / n, qx / n, qy / n, qz / n
    r = np.stack([
        1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
        2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
        2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)], -1)
    return r.reshape(np.shape(qw) + (3, 3))


def init_backbone(cfg: IpaConfig, seed: int, layer: int):
    w = gaussian_tensor(Rng(seed + 1000 + layer), (cfg.d_in, 6), 0.1 / math.sqrt(cfg.d_in))
    return {"w": w, "b": np.zeros(6)}


def init_trunk(cfg: IpaConfig, n_layers: int, seed: int):
    return ([init_weights(cfg, seed + l) for l in range(n_layers)],
            [init_backbone(cfg, seed, l) for l in range(n_layers)])


def backbone_update(s, rot, trans, mask, bb):
    u = s @ bb["w"] + bb["b"]
    dR = quat_to_rot(np.ones(len(s)), u[:, 0], u[:, 1], u[:, 2])
    new_rot = np.einsum("lab,lbc->lac", rot, dR)
    new_t = np.einsum("lab,lb->la", rot, u[:, 3:6]) + trans
    m = np.asarray(mask, bool)[:, None]
    return np.where(m[..., None], new_rot, rot), np.where(m, new_t, trans)


def trunk_forward(s, z1, z2, rot, trans, mask, cfg: IpaConfig, layers, backbones):
    mask = np.ones(s.shape[0], bool) if mask is None else np.asarray(mask, bool)
    for w, bb in zip(layers, backbones):
        s = s + flash_ipa_forward(s, z1, z2, rot, trans, mask, cfg, w)
        rot, trans = backbone_update(s, rot, trans, mask, bb)
    return s, rot, trans



# --------------------------------------------------------------- pair-factor producer
def positional_encoding(offsets, dim):
    """proj/src/pair_features.cpp:66-81: [sin(x f_p), cos(x f_p)] with f_p = 10000^(-2p/dim)."""
    if dim < 2 or dim % 2:
        raise ValueError("positional encoding width must be even")
    x = np.asarray(offsets, np.float64)[:, None]
    p = np.arange(dim // 2)
    freq = np.array([math.pow(10000.0, -(2.0 * q) / dim) for q in p])
    out = np.empty((len(offsets), dim))
    out[:, 0::2] = np.sin(x * freq)
    out[:, 1::2] = np.cos(x * freq)
    return out


def knn_distogram(trans, k=20, n_bins=22, d_min=2.0, d_max=22.0, pe_dim=16):
    """proj/src/pair_features.cpp:10-64: k nearest other residues (Euclidean, ties to the lower
    index), one-hot distance bins (clipped into the end bins) + encoding of the offset j - i."""
    trans = np.asarray(trans, np.float64)
    L = trans.shape[0]
    if L < 2 or not 1 <= k <= L - 1 or n_bins < 2 or not d_min < d_max or pe_dim % 2:
        raise ValueError("invalid distogram spec")
    width = (d_max - d_min) / n_bins
    out = np.zeros((L, k, n_bins + pe_dim))
    for i in range(L):
        d = trans - trans[i]
        dist = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])
        idx = np.array([j for j in range(L) if j != i])
        order = idx[np.lexsort((idx, dist[idx]))][:k]  # distance, then lower index
        rel = np.maximum((dist[order] - d_min) / width, 0.0)
        bins = np.minimum(rel.astype(np.int64), n_bins - 1)
        out[i, np.arange(k), bins] = 1.0
        out[i, :, n_bins:] = positional_encoding(order - i, pe_dim)
    return out


def build_factors(features, r, d_z, w1, w2):
    """proj/src/pair_features.cpp:83-97."""
    L = features.shape[0]
    return (features @ w1).reshape(L, r, d_z), (features @ w2).reshape(L, r, d_z)
