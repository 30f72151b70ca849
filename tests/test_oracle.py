"""CPU: the numpy oracle restatement pinned against fixtures produced by the reference itself
(tests/golden/, written by oracle/gen_golden.py from the reference compiled from its sources)."""

import os

import numpy as np
import pytest

from oracle import fipa_oracle as fo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SHAPES = {
    "tiny": dict(d_in=32, d_z=4, heads=2, c=8, n_query=2, n_value=2, rank=2),
    "h1_r1_q1_v1": dict(d_in=12, d_z=4, heads=1, c=5, n_query=1, n_value=1, rank=1),
    "h4_r2_q4_v8": dict(d_in=12, d_z=4, heads=4, c=5, n_query=4, n_value=8, rank=2),
    "main": dict(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2),
}


def cfg_of(name, precision="f64"):
    return fo.IpaConfig(**SHAPES[name], precision=precision, enforce_head_cap=False)


def test_rng_stream_is_bit_identical_to_reference():
    g = np.load(os.path.join(GOLD, "rng.npz"))
    assert np.array_equal(fo.Rng(3).gaussians(1001), g["gauss_seed3"])
    r = fo.Rng(3)
    assert np.array_equal(np.array([r.gaussian() for _ in range(1001)]), g["gauss_seed3"])
    rot, trans = fo.random_frames(fo.Rng(5), 10, 1.0)
    assert np.array_equal(rot, g["frames_seed5_rot"]) and np.array_equal(trans, g["frames_seed5_trans"])


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_init_weights_bit_identical(name, precision):
    """IpaWeights::init (proj/src/ipa.cpp:172-193) draw order and scales."""
    g = np.load(os.path.join(GOLD, "weights_seed7.npz"))
    w = fo.init_weights(cfg_of(name, precision), 7)
    for n in fo.WEIGHT_NAMES:
        if name == "main":
            assert np.array_equal(w[n].ravel()[:64], g[f"{name}/{precision}/{n}/head"])
            assert np.sum(w[n]) == float(g[f"{name}/{precision}/{n}/sum"])
        else:
            assert np.array_equal(w[n], g[f"{name}/{precision}/{n}"]), n
    assert w["w_l"] == float(g[f"{name}/{precision}/w_l"])
    assert w["w_c"] == float(g[f"{name}/{precision}/w_c"])


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("tag", ["plain", "masked", "far"])
def test_forward_restatement_matches_reference(name, tag):
    g = np.load(os.path.join(GOLD, f"forward_{name}.npz"))
    cfg = cfg_of(name)
    w = fo.init_weights(cfg, 7)
    args = [g[f"{tag}/{k}"] for k in ("s", "z1", "z2", "rot", "trans", "mask")]
    out = fo.flash_ipa_forward(*args, cfg, w)
    assert fo.rel_dev(g[f"{tag}/flash"], out) < 1e-12
    quad = fo.reference_forward(*args, cfg, w)
    assert fo.rel_dev(g[f"{tag}/reference"], quad) < 1e-12
    # the reference's own flash == quadratic guarantee (proj/tests/test_flash_ipa.cpp:170-202)
    assert fo.rel_dev(g[f"{tag}/reference"], g[f"{tag}/flash"]) < 1e-10
    mask = g[f"{tag}/mask"].astype(bool)
    assert np.all(out[~mask] == 0.0)


@pytest.mark.parametrize("name", ["tiny", "h1_r1_q1_v1", "h4_r2_q4_v8"])
def test_lifted_rows_match_reference(name):
    g = np.load(os.path.join(GOLD, f"forward_{name}.npz"))
    cfg = cfg_of(name)
    w = fo.init_weights(cfg, 7)
    q, k, v = fo.lift_qkv(*[g[f"plain/{x}"] for x in ("s", "z1", "z2", "rot", "trans")], cfg, w)
    assert fo.rel_dev(g["plain/q_hat"], q) < 1e-13
    assert fo.rel_dev(g["plain/k_hat"], k) < 1e-13
    assert fo.rel_dev(g["plain/v_hat"], v) < 1e-13


def test_lifted_logit_identity_and_negative_control():
    """<q_hat_i, k_hat_j> equals the quadratic logit; swapping the ones/norm segments breaks it
    (proj/tests/test_flash_ipa.cpp:101-168)."""
    cfg = cfg_of("h4_r2_q4_v8")
    w = fo.init_weights(cfg, 3)
    p = fo.make_problem(cfg, 11, seed=4)
    q, k, _ = fo.lift_qkv(p.s, p.z1, p.z2, p.rot, p.trans, cfg, w)
    qq, kk, _, qp, kp, _ = fo.project_inputs(p.s, cfg, w)
    gq = fo.apply(p.rot[None, :, None], p.trans[None, :, None], qp)
    gk = fo.apply(p.rot[None, :, None], p.trans[None, :, None], kp)
    z = np.einsum("ird,jrd->ijd", p.z1, p.z2)
    bias = np.einsum("hd,ijd->hij", w["w_bias"], z)
    dist = ((gq[:, :, None] - gk[:, None, :]) ** 2).sum((-1, -2))
    gamma = fo.softplus(w["gamma_raw"])
    logits = w["w_l"] * (np.einsum("hic,hjc->hij", qq, kk) / np.sqrt(cfg.c)
                         + bias - (0.5 * gamma * w["w_c"])[:, None, None] * dist)
    lifted = np.einsum("hid,hjd->hij", q, k)
    assert fo.rel_dev(logits, lifted) < 1e-12
    c, n = cfg.c, cfg.n_query
    q_bad = q.copy()
    q_bad[..., c + 3 * n:c + 4 * n], q_bad[..., c + 4 * n:c + 5 * n] = q[..., c + 4 * n:c + 5 * n], q[..., c + 3 * n:c + 4 * n]
    assert fo.rel_dev(logits, np.einsum("hid,hjd->hij", q_bad, k)) > 1e-3


def test_oracle_invariance_under_global_motion():
    cfg = cfg_of("tiny")
    w = fo.init_weights(cfg, 5)
    p = fo.make_problem(cfg, 19, seed=9, translation_scale=5.0)
    g_rot, g_t = fo.random_rototranslation(fo.Rng(77), 10.0)
    rot2 = np.einsum("ab,ibc->iac", g_rot, p.rot)
    trans2 = p.trans @ g_rot.T + g_t
    a = fo.flash_ipa_forward(p.s, p.z1, p.z2, p.rot, p.trans, None, cfg, w)
    b = fo.flash_ipa_forward(p.s, p.z1, p.z2, rot2, trans2, None, cfg, w)
    assert fo.rel_dev(a, b) < 1e-12


def test_bf16_rounding_helper():
    x = np.array([1.0, 1.0 + 2 ** -7, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 3.14159, -2.5e-3])
    r = fo.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 + 2 ** -7          # representable: unchanged
    assert r[2] == 1.0 and r[3] == 1.0 + 2 ** -6           # ties round to even
    assert np.all(fo.round_bf16(r) == r)                   # idempotent
    assert np.max(np.abs(r - x) / np.abs(x)) <= 2 ** -8


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                                                    "libfipa_ref.so")), reason="reference oracle not built")
def test_live_reference_cross_check():
    from oracle import ref

    cfg = cfg_of("h4_r2_q4_v8")
    w = ref.init_weights(cfg, 21)
    p = fo.make_problem(cfg, 31, seed=22, mask_frac=0.2)
    a = ref.flash_forward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, p.mask, tile_rows=7, tile_cols=5, threads=3)
    b = fo.flash_ipa_forward(p.s, p.z1, p.z2, p.rot, p.trans, p.mask, cfg, fo.init_weights(cfg, 21))
    assert fo.rel_dev(a, b) < 1e-12


def test_backward_matches_reference_finite_differences():
    """The float64 backward restatement (fipa_oracle.flash_ipa_backward) against central finite
    differences of the reference's own flash_ipa_forward (fixture from oracle/gen_golden.py),
    with a masked residue, non-unit gamma and a nonzero output bias."""
    g = np.load(os.path.join(GOLD, "backward_fd.npz"))
    from oracle.gen_golden import FD_SHAPE

    cfg = fo.IpaConfig(**FD_SHAPE, enforce_head_cap=False)
    w = {n: g[f"w/{n}"] for n in fo.WEIGHT_NAMES}
    w["w_l"] = np.sqrt(1.0 / 3.0)
    w["w_c"] = np.sqrt(2.0 / (9.0 * cfg.n_query))
    ins = {k: g[f"in/{k}"] for k in ("s", "z1", "z2", "rot", "trans")}
    got = fo.flash_ipa_backward(ins["s"], ins["z1"], ins["z2"], ins["rot"], ins["trans"],
                                g["in/mask"], cfg, w, g["in/dout"])
    for name in list(ins) + list(fo.WEIGHT_NAMES):
        assert fo.rel_dev(g[f"grad/{name}"], got[name]) < 1e-7, name
    # masked residue: no gradient reaches its inputs
    m = ~g["in/mask"].astype(bool)
    for name in ("s", "z1", "z2", "rot", "trans"):
        assert np.abs(got[name][m]).max() < 1e-12, name


def test_backward_all_masked_is_zero():
    cfg = cfg_of("tiny")
    w = fo.init_weights(cfg, 1)
    p = fo.make_problem(cfg, 5, 3)
    got = fo.flash_ipa_backward(p.s, p.z1, p.z2, p.rot, p.trans, np.zeros(5, bool), cfg, w,
                                np.ones((5, cfg.d_in)))
    assert all(np.abs(v).max() == 0 for v in got.values())
