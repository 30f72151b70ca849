"""ORACLE / TEST INFRASTRUCTURE ONLY: regenerate tests/golden/ from the compiled reference.

The reference ships no golden vectors, so the fixtures are produced by the
reference itself: oracle/_ref/libfipa_ref.so, compiled by oracle/Makefile from the unmodified
sources under /root/reference/proj/src.  Run here (the reference is not on the GPU box):

    make -C oracle && python -m oracle.gen_golden
"""

from __future__ import annotations

import os

import numpy as np

from . import ref
from .fipa_oracle import IpaConfig, WEIGHT_NAMES, make_problem

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

TINY = dict(d_in=32, d_z=4, heads=2, c=8, n_query=2, n_value=2, rank=2)
MAIN = dict(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2)
# proj/tests/test_flash_ipa.cpp:30-47 problem family (d_in 12, d_z 4, c 5) at several H/r/N
SHAPES = {
    "tiny": TINY,
    "h1_r1_q1_v1": dict(d_in=12, d_z=4, heads=1, c=5, n_query=1, n_value=1, rank=1),
    "h4_r2_q4_v8": dict(d_in=12, d_z=4, heads=4, c=5, n_query=4, n_value=8, rank=2),
    "main": MAIN,
}


def cfg_of(shape, precision="f64"):
    return IpaConfig(**shape, precision=precision, enforce_head_cap=False)


def main():
    os.makedirs(OUT, exist_ok=True)
    # RNG streams: gaussian draws and random rigid frames (proj/src/rng.cpp, geometry.cpp:107-132)
    rot, trans = ref.random_frames(5, 10, 1.0)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), gauss_seed3=ref.gaussian(3, 1001),
                        frames_seed5_rot=rot, frames_seed5_trans=trans)

    # Weights: full tensors for the small shapes, checksums + heads of each tensor for MAIN.
    wfix = {}
    for name, shape in SHAPES.items():
        for prec in ("f64", "f32"):
            w = ref.init_weights(cfg_of(shape, prec), 7)
            for n in WEIGHT_NAMES:
                if name == "main":
                    wfix[f"{name}/{prec}/{n}/sum"] = np.array(np.sum(w[n]))
                    wfix[f"{name}/{prec}/{n}/head"] = w[n].ravel()[:64].copy()
                else:
                    wfix[f"{name}/{prec}/{n}"] = w[n]
            wfix[f"{name}/{prec}/w_l"] = np.array(w["w_l"])
            wfix[f"{name}/{prec}/w_c"] = np.array(w["w_c"])
    np.savez_compressed(os.path.join(OUT, "weights_seed7.npz"), **wfix)

    # Weights file written by the reference (proj/src/model_io.cpp:121-141).
    ref.save_weights(cfg_of(TINY), ref.init_weights(cfg_of(TINY), 11), os.path.join(OUT, "tiny_seed11.fipa"))
    ref.save_weights(cfg_of(TINY, "f32"), ref.init_weights(cfg_of(TINY, "f32"), 11),
                     os.path.join(OUT, "tiny_f32_seed11.fipa"))

    # Forward outputs of the reference flash path and quadratic path at f64 (and flash at f32).
    for name, shape in SHAPES.items():
        L = 48 if name == "main" else 23
        cfg = cfg_of(shape)
        w = ref.init_weights(cfg, 7)
        rec = {}
        for tag, mask_frac, scale in (("plain", 0.0, 1.0), ("masked", 0.25, 1.0), ("far", 0.0, 30.0)):
            p = make_problem(cfg, L, seed=101, translation_scale=scale, mask_frac=mask_frac)
            rec[f"{tag}/s"], rec[f"{tag}/z1"], rec[f"{tag}/z2"] = p.s, p.z1, p.z2
            rec[f"{tag}/rot"], rec[f"{tag}/trans"], rec[f"{tag}/mask"] = p.rot, p.trans, p.mask
            rec[f"{tag}/flash"] = ref.flash_forward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, p.mask)
            rec[f"{tag}/reference"] = ref.reference_forward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, p.mask)
            if tag == "plain" and name != "main":
                q, k, v = ref.lift(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans)
                rec[f"{tag}/q_hat"], rec[f"{tag}/k_hat"], rec[f"{tag}/v_hat"] = q, k, v
                cf = cfg_of(shape, "f32")
                wf = ref.init_weights(cf, 7)
                rec[f"{tag}/flash_f32"] = ref.flash_forward(cf, wf, p.s, p.z1, p.z2, p.rot, p.trans, p.mask)
        np.savez_compressed(os.path.join(OUT, f"forward_{name}.npz"), **rec)

    # Backward: the reference has no autodiff (proj/SPEC.md:8), so its gradient is pinned by
    # central finite differences of the reference's own flash_ipa_forward (f64).
    np.savez_compressed(os.path.join(OUT, "backward_fd.npz"), **backward_fd_fixture())
    print("golden fixtures written to", OUT)


FD_SHAPE = dict(d_in=12, d_z=3, heads=2, c=4, n_query=2, n_value=3, rank=2)
FD_EPS = 1e-6


def backward_fd_fixture():
    cfg = cfg_of(FD_SHAPE)
    w = ref.init_weights(cfg, 3)
    rng = np.random.default_rng(0)
    w["b_out"] = rng.standard_normal(w["b_out"].shape)
    w["gamma_raw"] = np.array([0.3, -0.7])
    L = 7
    p = make_problem(cfg, L, seed=11, translation_scale=2.0)
    mask = np.ones(L, bool)
    mask[2] = False
    dout = rng.standard_normal((L, cfg.d_in))
    inputs = dict(s=p.s, z1=p.z1, z2=p.z2, rot=p.rot, trans=p.trans)
    rec = {f"in/{k}": v for k, v in inputs.items()}
    rec["in/mask"], rec["in/dout"] = mask, dout
    rec.update({f"w/{n}": w[n] for n in WEIGHT_NAMES})

    def loss(name, x):
        a, ww = dict(inputs), dict(w)
        (a if name in a else ww)[name] = x
        out = ref.flash_forward(cfg, ww, a["s"], a["z1"], a["z2"], a["rot"], a["trans"], mask)
        return float((out * dout).sum())

    for name in list(inputs) + list(WEIGHT_NAMES):
        x = np.array(inputs[name] if name in inputs else w[name], dtype=np.float64)
        fd = np.zeros_like(x)
        for idx in np.ndindex(x.shape):
            xp, xm = x.copy(), x.copy()
            xp[idx] += FD_EPS
            xm[idx] -= FD_EPS
            fd[idx] = (loss(name, xp) - loss(name, xm)) / (2 * FD_EPS)
        rec[f"grad/{name}"] = fd
    return rec


if __name__ == "__main__":
    main()
