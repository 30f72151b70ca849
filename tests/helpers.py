"""Shared test helpers: problem generation, oracle runs, GPU runs through the C ABI.

The oracle (oracle/fipa_oracle.py) is the checker only; GPU results always come from the
native library (libfipa_b200.so) through the Model binding.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import fipa_oracle as fo

MAIN = dict(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2)  # north-star shape
TINY = dict(d_in=32, d_z=4, heads=2, c=8, n_query=2, n_value=2, rank=2)  # reference Model() default

BF16_TOL = 2e-2  # north_star: bf16 inputs, fp32 accumulation
F32_TOL = 1e-4  # north_star: fp32 path


def oracle_cfg(shape: dict, precision="f64") -> fo.IpaConfig:
    return fo.IpaConfig(**shape, precision=precision, enforce_head_cap=False)


def make_batch(shape, B, L, seed, translation_scale=1.0, mask_frac=0.0, bf16=False):
    """B independent reference-style problems, stacked on a leading axis."""
    cfg = oracle_cfg(shape)
    probs = [fo.make_problem(cfg, L, seed + 17 * b, translation_scale, mask_frac) for b in range(B)]
    out = {k: np.stack([getattr(p, k) for p in probs]) for k in ("s", "z1", "z2", "rot", "trans", "mask")}
    if bf16:
        for k in ("s", "z1", "z2"):
            out[k] = fo.round_bf16(out[k])
    return out


def oracle_weights_for(model, precision):
    """The weights the GPU path actually computes with, as float64 for the oracle."""
    w = dict(model.weights())
    if precision == "bf16":
        for n in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp", "w_out"):
            w[n] = fo.round_bf16(w[n])
        for n in ("w_bias", "b_out"):
            w[n] = fo.round_f32(w[n])
    return w


def oracle_forward(shape, w, batch, return_intermediates=False):
    cfg = oracle_cfg(shape)
    outs, inters = [], []
    for b in range(batch["s"].shape[0]):
        r = fo.flash_ipa_forward(batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b],
                                 batch["trans"][b], batch["mask"][b], cfg, w,
                                 return_intermediates=return_intermediates)
        if return_intermediates:
            outs.append(r[0])
            inters.append(r[1])
        else:
            outs.append(r)
    return (np.stack(outs), inters) if return_intermediates else np.stack(outs)


def rel_dev(ref, got):
    return fo.rel_dev(ref, got)


def random_rigid(seed, scale=10.0):
    rng = fo.Rng(seed)
    return fo.random_rototranslation(rng, scale)


def move_frames(batch, g_rot, g_trans):
    """Global rigid motion g . T_i for every frame (proj/src/bench.cpp:56-62)."""
    out = dict(batch)
    out["rot"] = np.einsum("ab,...bc->...ac", g_rot, batch["rot"])
    out["trans"] = np.einsum("ab,...b->...a", g_rot, batch["trans"]) + g_trans
    return out


# ------------------------------------------------------------------ GPU side
def gpu_forward_device(model, batch):
    """Run fipa_layer_forward over torch-owned device buffers; returns (out, workspace, layout)."""
    import torch

    dev = torch.device("cuda:0")
    B, L = batch["s"].shape[:2]
    t = {k: torch.from_numpy(np.ascontiguousarray(batch[k], dtype=np.float32)).to(dev)
         for k in ("s", "z1", "z2", "rot", "trans")}
    mask = torch.from_numpy(np.ascontiguousarray(batch["mask"], dtype=np.uint8)).to(dev)
    out = torch.empty((B, L, model.config["d_in"]), dtype=torch.float32, device=dev)
    nbytes = model.workspace_size(B, L)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    model.forward_device(B, L, t["s"].data_ptr(), t["z1"].data_ptr(), t["z2"].data_ptr(),
                         t["rot"].data_ptr(), t["trans"].data_ptr(), mask.data_ptr(), out.data_ptr(),
                         ws.data_ptr(), nbytes, stream.cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), ws, model.workspace_layout(B, L)


def ws_view(ws, offset, count, dtype):
    """Typed float64 numpy copy of `count` elements at byte `offset` of a torch uint8 workspace."""
    import torch

    nbytes = count * (2 if dtype == "bf16" else 4)
    raw = ws[offset:offset + nbytes]
    if dtype == "bf16":
        return raw.view(torch.bfloat16).float().cpu().numpy().astype(np.float64)
    return raw.view(torch.float32).cpu().numpy().astype(np.float64)


def expected_lifted(shape, w, batch, b):
    """Oracle view of sample b in the B200 layout.

    Returns (logits, v_parts, cb):
      logits [H, L, L]  the reference attention logits <q_hat_i, k_hat_j> (natural units,
                        masked keys excluded later by the caller),
      v_parts [H, L, c + r d_z + 3Nv + 3]  [v | z2 | R_j v_p | t_j (recentred)],
      cb [H, L]  -g/2 sum_p |T_j k_p|^2 with -inf for masked keys.
    """
    cfg = oracle_cfg(shape)
    s, z1, z2, rot, trans = (batch[k][b] for k in ("s", "z1", "z2", "rot", "trans"))
    valid = batch["mask"][b].astype(bool)
    trans_c = trans - (trans[valid].mean(0) if valid.any() else 0.0)
    qh, kh, _ = fo.lift_qkv(s, z1, z2, rot, trans, cfg, w)
    logits = np.einsum("hid,hjd->hij", qh, kh)
    q, k, v, qp, kp, vp = fo.project_inputs(s, cfg, w)
    H, L = cfg.heads, s.shape[0]
    gamma = fo.softplus(w["gamma_raw"])
    g = (gamma * w["w_l"] * w["w_c"])[:, None]
    gk = fo.apply(rot[None, :, None], trans_c[None, :, None], kp)
    rv = np.einsum("lab,hlpb->hlpa", rot, vp).reshape(H, L, -1)
    z2f = np.broadcast_to(z2.reshape(1, L, -1), (H, L, cfg.rank * cfg.d_z))
    tt = np.broadcast_to(trans_c[None], (H, L, 3))
    v_parts = np.concatenate([v, z2f, rv, tt], -1)
    cb = -0.5 * g * (gk ** 2).sum((-1, -2))
    cb = np.where(valid[None], cb, -np.inf)
    return logits, v_parts, cb


def oracle_backward(shape, w, batch, dout):
    """Per-sample oracle gradients (fipa_oracle.flash_ipa_backward), stacked on the batch axis."""
    cfg = oracle_cfg(shape)
    res = []
    for b in range(batch["s"].shape[0]):
        res.append(fo.flash_ipa_backward(batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b],
                                         batch["trans"][b], batch["mask"][b], cfg, w, dout[b]))
    out = {k: np.stack([r[k] for r in res]) for k in ("s", "z1", "z2", "rot", "trans")}
    for n in fo.WEIGHT_NAMES:
        out[n] = sum(r[n] for r in res)
    return out


def emulated_backward(shape, w, batch, dout):
    """Oracle-equivalent forward output + gradients at large L: tests/bwd_emulation.py run with
    EXACT_SPLIT (the lifted-row restatement of fipa_oracle.flash_ipa_backward, equal to it within
    1e-14 -- tests/test_bwd_layout.py pins it on the CPU), query-blocked BLAS matmuls and O(L) memory
    per block, so L = 4096 finishes in seconds where the dense oracle needs O(L^2 d_z) memory.
    Returns (out [B,L,d_in], grads stacked like oracle_backward)."""
    import bwd_emulation as be

    cfg = oracle_cfg(shape)
    prev = be.EXACT_SPLIT
    be.EXACT_SPLIT = True
    try:
        outs, res = [], []
        for b in range(batch["s"].shape[0]):
            args = [batch[k][b] for k in ("s", "z1", "z2", "rot", "trans", "mask")]
            g, inter = be.backward(cfg, w, *args, dout[b])
            m = np.asarray(batch["mask"][b], bool)
            out = inter["feat"] @ w["w_out"] + w["b_out"] if inter else np.zeros_like(batch["s"][b])
            outs.append(np.where(m[:, None], out, 0.0))
            res.append(g)
    finally:
        be.EXACT_SPLIT = prev
    grads = {k: np.stack([r[k] for r in res]) for k in ("s", "z1", "z2", "rot", "trans")}
    for n in fo.WEIGHT_NAMES:
        grads[n] = sum(r[n] for r in res)
    return np.stack(outs), grads


def emulated_forward(cfg, w, s, z1, z2, rot, trans, mask):
    """Oracle-equivalent layer forward of one sample at large L (tests/bwd_emulation.py with
    EXACT_SPLIT: the lifted-row restatement of fipa_oracle.flash_ipa_forward, query-blocked)."""
    import bwd_emulation as be

    mask = np.asarray(mask, bool)
    if not mask.any():
        return np.zeros_like(s)
    prev = be.EXACT_SPLIT
    be.EXACT_SPLIT = True
    try:
        trans_c = trans - trans[mask].mean(0)
        pk = be.pack(cfg, w, s, z1, z2, rot, trans_c, mask)
        o_hat, _ = be.attention(pk["q_hat"], pk["k_hat"], pk["v_hat"], s.shape[0])
        feat, _ = be.epilogue(cfg, o_hat, z1, rot, trans_c)
    finally:
        be.EXACT_SPLIT = prev
    out = feat @ w["w_out"] + w["b_out"]
    return np.where(mask[:, None], out, 0.0)


def emulated_trunk(cfg, layers, backbones, s, z1, z2, rot, trans, mask, layer_input=None):
    """fipa_oracle.trunk_forward over emulated_forward; layer_input (e.g. round_bf16) is applied
    to s where each layer reads it (the device casts a layer's input to bf16 for its projection
    GEMM; the residual stream stays fp32)."""
    mask = np.asarray(mask, bool)
    for w, bb in zip(layers, backbones):
        x = layer_input(s) if layer_input is not None else s
        s = s + emulated_forward(cfg, w, x, z1, z2, rot, trans, mask)
        rot, trans = fo.backbone_update(s, rot, trans, mask, bb)
    return s, rot, trans


def gpu_train_device(model, batch, dout):
    """forward_train + backward through the C ABI over torch-owned device buffers.
    Returns (out, grads, workspace, layouts)."""
    import torch

    dev = torch.device("cuda:0")
    B, L = batch["s"].shape[:2]
    t = {k: torch.from_numpy(np.ascontiguousarray(batch[k], dtype=np.float32)).to(dev)
         for k in ("s", "z1", "z2", "rot", "trans")}
    mask = torch.from_numpy(np.ascontiguousarray(batch["mask"], dtype=np.uint8)).to(dev)
    dt = torch.from_numpy(np.ascontiguousarray(dout, dtype=np.float32)).to(dev)
    out = torch.empty((B, L, model.config["d_in"]), dtype=torch.float32, device=dev)
    nbytes = model.train_workspace_size(B, L)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    g = {k: torch.full_like(v, float("nan")) for k, v in t.items()}
    gw = torch.full((model.num_weights(),), float("nan"), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    p = {k: v.data_ptr() for k, v in t.items()}
    model.forward_train_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], mask.data_ptr(),
                               out.data_ptr(), ws.data_ptr(), nbytes, st)
    model.backward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], mask.data_ptr(),
                          dt.data_ptr(), g["s"].data_ptr(), g["z1"].data_ptr(), g["z2"].data_ptr(),
                          g["rot"].data_ptr(), g["trans"].data_ptr(), gw.data_ptr(), ws.data_ptr(), nbytes, st)
    torch.cuda.synchronize()
    grads = {k: v.cpu().numpy().astype(np.float64) for k, v in g.items()}
    flat = gw.cpu().numpy().astype(np.float64)
    sh = fo.weight_shapes(oracle_cfg({k: model.config[k] for k in MAIN}))
    o = 0
    for n in fo.WEIGHT_NAMES:
        size = int(np.prod(sh[n]))
        grads[n] = flat[o:o + size].reshape(sh[n])
        o += size
    return (out.cpu().numpy().astype(np.float64), grads, ws,
            (model.workspace_layout(B, L), model.train_workspace_layout(B, L)))
