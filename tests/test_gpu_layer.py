"""GPU parity tests: the sm_100a kernels (through the C ABI) against the oracle.

Tolerances are the north_star's: max relative error (max|a-b| / max|ref|,
proj/tests/test_support.hpp:31-34) <= 2e-2 for bf16 inputs with fp32 accumulation and
<= 1e-4 for the fp32 path, against the float64 oracle fed the same (rounded) inputs.
"""

import numpy as np
import pytest

from helpers import (BF16_TOL, F32_TOL, MAIN, TINY, expected_lifted, gpu_forward_device,
                     make_batch, move_frames, oracle_cfg, oracle_forward, oracle_weights_for,
                     random_rigid, rel_dev, ws_view)
from oracle import fipa_oracle as fo

pytestmark = pytest.mark.gpu


def _model(fipa, shape, precision, seed=0):
    return fipa.Model(**shape, precision=precision, seed=seed, enforce_head_cap=False)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
def test_stage_by_stage_main_shape(fipa, precision):
    """Every intermediate of the north-star shape (c_s 256, c_z 128, H 8, 8/12 points, rank 2)
    on a ragged length with masked rows."""
    B, L = 2, 200
    bf = precision == "bf16"
    model = _model(fipa, MAIN, precision, seed=5)
    w = oracle_weights_for(model, precision)
    batch = make_batch(MAIN, B, L, seed=1000, mask_frac=0.1, bf16=bf)
    batch["mask"][0, :] = True
    out, ws, (off, dims) = gpu_forward_device(model, batch)
    n_proj, dqk_pad, dv_pad, nfeat = dims
    H = MAIN["heads"]
    el = "bf16" if bf else "f32"
    cfg = oracle_cfg(MAIN)

    # projection GEMM: s . W_fused (fp32 accumulation)
    proj = ws_view(ws, off[2], B * L * n_proj, "f32").reshape(B, L, n_proj)
    wf = np.concatenate([w[n] for n in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp")], axis=1)
    # the fused bf16 projection+pack kernel keeps only the point columns (what the backward reads)
    pts0 = 3 * MAIN["heads"] * MAIN["c"] if bf else 0
    assert rel_dev((batch["s"] @ wf)[..., pts0:], proj[..., pts0:]) < 1e-5

    qh = ws_view(ws, off[3], B * H * L * dqk_pad, el).reshape(B, H, L, dqk_pad)
    kh = ws_view(ws, off[4], B * H * L * dqk_pad, el).reshape(B, H, L, dqk_pad)
    vh = ws_view(ws, off[5], B * H * L * dv_pad, el).reshape(B, H, L, dv_pad)
    cb = ws_view(ws, off[6], B * H * L, "f32").reshape(B, H, L)
    L2E = 1.0 / np.log(2.0)
    for b in range(B):
        elog, ev, ecb = expected_lifted(MAIN, w, batch, b)
        valid = batch["mask"][b].astype(bool)
        # q_hat . k_hat must equal log2(e) * (reference logit) up to a per-row constant
        # (the dropped |T_i q_p|^2 term), and masked keys must sit at <= -1e29.
        s_gpu = np.einsum("hid,hjd->hij", qh[b], kh[b])
        assert np.all(s_gpu[:, :, ~valid] < -1e29)
        d_gpu = s_gpu[:, :, valid] - s_gpu[:, :, valid][:, :, :1]
        d_ref = L2E * (elog[:, :, valid] - elog[:, :, valid][:, :, :1])
        assert rel_dev(d_ref, d_gpu) < (4e-3 if bf else 1e-6)
        # v_hat = [v | z2 | t hi | t lo | R_j v_p | 0]   (pack.cu)
        npair = MAIN["c"] + MAIN["rank"] * MAIN["d_z"]
        npts = 3 * MAIN["n_value"]
        assert rel_dev(ev[..., :npair], vh[b, :, :, :npair]) < (8e-3 if bf else 1e-6)
        t_sum = vh[b, :, :, npair:npair + 3] + vh[b, :, :, npair + 3:npair + 6]
        assert rel_dev(ev[..., -3:], t_sum) < (1e-5 if bf else 1e-6)
        assert rel_dev(ev[..., npair:npair + npts], vh[b, :, :, npair + 6:npair + 6 + npts]) < (8e-3 if bf else 1e-6)
        assert np.all(vh[b, :, :, npair + 6 + npts:] == 0)
        fin = np.isfinite(ecb)
        assert np.array_equal(fin, np.isfinite(cb[b]))
        assert rel_dev(ecb[fin], cb[b][fin]) < 1e-5

    ref, inter = oracle_forward(MAIN, w, batch, return_intermediates=True)
    feat = ws_view(ws, off[8], B * L * nfeat, el).reshape(B, L, nfeat)
    tol = BF16_TOL if bf else F32_TOL
    for b in range(B):
        valid = batch["mask"][b].astype(bool)
        assert rel_dev(inter[b]["feat"][valid], feat[b][valid]) < tol
    assert rel_dev(ref, out) < tol
    assert np.all(out[~batch["mask"].astype(bool)] == 0.0)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
@pytest.mark.parametrize("L", [1, 7, 64, 129, 333])
def test_layer_parity_lengths(fipa, precision, L):
    """Host-buffer path (Model.flash, the reference calling convention) across ragged lengths."""
    bf = precision == "bf16"
    model = _model(fipa, MAIN, precision, seed=11)
    w = oracle_weights_for(model, precision)
    batch = make_batch(MAIN, 1, L, seed=2000 + L, bf16=bf)
    got = model.flash(batch["s"][0], batch["z1"][0], batch["z2"][0], batch["rot"][0], batch["trans"][0])
    ref = oracle_forward(MAIN, w, batch)[0]
    assert got.shape == (L, MAIN["d_in"])
    assert rel_dev(ref, got) < (BF16_TOL if bf else F32_TOL)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
@pytest.mark.parametrize("shape", [TINY, dict(d_in=12, d_z=4, heads=4, c=5, n_query=4, n_value=8, rank=1),
                                   dict(d_in=12, d_z=4, heads=1, c=5, n_query=1, n_value=1, rank=2)])
def test_small_shapes(fipa, precision, shape):
    """Reference test shapes (proj/tests/test_flash_ipa.cpp:170-202) incl. odd widths."""
    bf = precision == "bf16"
    model = _model(fipa, shape, precision, seed=4)
    w = oracle_weights_for(model, precision)
    batch = make_batch(shape, 3, 37, seed=77, mask_frac=0.2, bf16=bf)
    got = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], mask=batch["mask"])
    ref = oracle_forward(shape, w, batch)
    assert rel_dev(ref, got) < (BF16_TOL if bf else F32_TOL)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
def test_masking_semantics(fipa, precision):
    """Masked rows are zero and ignored; an all-masked sample is all zeros
    (proj/src/flash_ipa.cpp:156-159, 213-216; proj/tests/test_flash_ipa.cpp:231-255)."""
    model = _model(fipa, MAIN, precision, seed=3)
    w = oracle_weights_for(model, precision)
    batch = make_batch(MAIN, 3, 96, seed=31, mask_frac=0.3, bf16=precision == "bf16")
    batch["mask"][2, :] = False
    got = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], mask=batch["mask"])
    m = batch["mask"].astype(bool)
    assert np.all(got[~m] == 0.0)
    assert np.all(got[2] == 0.0)
    ref = oracle_forward(MAIN, w, batch)
    assert rel_dev(ref, got) < (BF16_TOL if precision == "bf16" else F32_TOL)
    # masking == deletion (proj/tests/test_attention_kernel.cpp:284-313)
    keep = np.where(m[0])[0]
    sub = {k: batch[k][:1, keep] for k in ("s", "z1", "z2", "rot", "trans")}
    got_sub = model.flash(sub["s"], sub["z1"], sub["z2"], sub["rot"], sub["trans"])
    assert rel_dev(got[0][keep], got_sub[0]) < (1e-2 if precision == "bf16" else 1e-5)


@pytest.mark.parametrize("precision,tol", [("bf16", BF16_TOL), ("f32", F32_TOL)])
@pytest.mark.parametrize("scale", [1.0, 30.0])
def test_se3_invariance(fipa, precision, tol, scale):
    """Outputs unchanged under a global rigid motion of all frames
    (proj/tests/test_flash_ipa.cpp:219-229; proj/src/bench.cpp:187-219)."""
    model = _model(fipa, MAIN, precision, seed=8)
    batch = make_batch(MAIN, 2, 150, seed=55, translation_scale=scale, bf16=precision == "bf16")
    g_rot, g_tr = random_rigid(123, 10.0)
    moved = move_frames(batch, g_rot, g_tr)
    a = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"])
    b = model.flash(moved["s"], moved["z1"], moved["z2"], moved["rot"], moved["trans"])
    assert rel_dev(a, b) < tol


def test_batch_is_independent_calls_and_tiles_ignored(fipa):
    model = _model(fipa, MAIN, "bf16", seed=9)
    batch = make_batch(MAIN, 3, 70, seed=90, bf16=True)
    got = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"])
    for b in range(3):
        one = model.flash(batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b], batch["trans"][b],
                          tile_rows=3, tile_cols=5, threads=4)
        assert np.array_equal(one, got[b])


def test_reference_model_defaults_roundtrip(fipa, tmp_path):
    """Reference smoke semantics (proj/tests/python/test_smoke.py) on the default tiny Model."""
    model = fipa.Model(seed=3)
    batch = make_batch(TINY, 1, 12, seed=1)
    args = [batch[k][0] for k in ("s", "z1", "z2", "rot", "trans")]
    w = oracle_weights_for(model, "f32")
    ref = oracle_forward(TINY, w, batch)[0]
    got = model.flash(*args)
    assert rel_dev(ref, got) < F32_TOL
    path = str(tmp_path / "w.fipa")
    model.save(path)
    other = fipa.Model(seed=999)
    other.load(path)
    assert np.array_equal(other.flash(*args), got)


@pytest.mark.parametrize("impl", ["1sm", "pair", "pass"])
def test_attention_kernels_agree(fipa, impl):
    """The tcgen05 attention kernels (single CTA, CTA pair, two-pass CTA pair) against the oracle at the
    north-star shape, ragged L with masked keys (Model.set_tuning(attn_impl=...) selects the kernel)."""
    model = _model(fipa, MAIN, "bf16", seed=21)
    model.set_tuning(attn_impl=impl)
    assert model.tuning()["attn_impl"] == impl
    w = oracle_weights_for(model, "bf16")
    batch = make_batch(MAIN, 2, 389, seed=4242, mask_frac=0.15, bf16=True)
    got = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], mask=batch["mask"])
    ref = oracle_forward(MAIN, w, batch)
    assert rel_dev(ref, got) < BF16_TOL


@pytest.mark.parametrize("L", [8192])
def test_long_sequence_properties(fipa, L):
    """Full-size properties without an O(L^2) oracle: a long single structure is finite, its
    output is invariant under a global rigid motion (reference bench.cpp:56-62 check) and a
    random subset of rows matches the oracle computed for those query rows only."""
    import torch

    model = _model(fipa, MAIN, "bf16", seed=13)
    batch = make_batch(MAIN, 1, L, seed=77, bf16=True)
    out, _, _ = gpu_forward_device(model, batch)
    assert np.all(np.isfinite(out))
    g_rot, g_t = random_rigid(5, scale=10.0)
    out2, _, _ = gpu_forward_device(model, move_frames(batch, g_rot, g_t))
    assert rel_dev(out, out2) < BF16_TOL
    # oracle on 64 sampled query rows against all L keys (dense over keys, cheap in float64)
    cfg = oracle_cfg(MAIN)
    w = oracle_weights_for(model, "bf16")
    rows = np.random.default_rng(0).choice(L, 64, replace=False)
    q, k, v = fo.lift_qkv(batch["s"][0], batch["z1"][0], batch["z2"][0], batch["rot"][0], batch["trans"][0], cfg, w)
    o = fo.flash_attention(q[:, rows], k, v)
    feat = fo.epilogue_features(o, batch["z1"][0][rows], batch["rot"][0][rows], batch["trans"][0][rows], cfg)
    ref = feat @ w["w_out"] + w["b_out"]
    assert rel_dev(ref, out[0][rows]) < BF16_TOL
    del torch


@pytest.mark.parametrize("rank", [3, 4])
@pytest.mark.parametrize("B,L,mask_frac", [(2, 200, 0.15), (1, 513, 0.0)])
def test_wide_rank_bf16(fipa, rank, B, L, mask_frac):
    """z_factor_rank 3-4 (lifted widths 560-704) on the tensor cores: the two-pass CTA-pair
    kernel (attn_fwd_pass.cu) against the oracle, ragged lengths and masked keys (BASELINE cfg5)."""
    shape = dict(MAIN, rank=rank)
    model = _model(fipa, shape, "bf16", seed=31 + rank)
    w = oracle_weights_for(model, "bf16")
    batch = make_batch(shape, B, L, seed=900 + rank * 10 + B, mask_frac=mask_frac, bf16=True)
    got = model.flash(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], mask=batch["mask"])
    ref = oracle_forward(shape, w, batch)
    assert rel_dev(ref, got) < BF16_TOL
    if mask_frac > 0:
        assert np.all(got[~batch["mask"].astype(bool)] == 0.0)


@pytest.mark.parametrize("rank", [3, 4])
def test_wide_rank_se3_invariance(fipa, rank):
    shape = dict(MAIN, rank=rank)
    model = _model(fipa, shape, "bf16", seed=5)
    batch = make_batch(shape, 1, 300, seed=61, bf16=True)
    args = (batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"])
    got = model.flash(*args)
    g_rot, g_t = random_rigid(9, scale=10.0)
    moved = move_frames(batch, g_rot, g_t)
    got2 = model.flash(moved["s"], moved["z1"], moved["z2"], moved["rot"], moved["trans"])
    assert rel_dev(got, got2) < BF16_TOL


def test_forward_bench_config_all_rows(fipa):
    """Inference forward at the benched workload (B=8, L=1024: ~3.5 waves of CTA pairs), every row
    of every sample against the oracle-equivalent blocked checker (helpers.emulated_backward)."""
    from helpers import emulated_backward

    model = _model(fipa, MAIN, "bf16", seed=23)
    w = oracle_weights_for(model, "bf16")
    batch = make_batch(MAIN, 8, 1024, seed=99, mask_frac=0.1, bf16=True)
    got, _, _ = gpu_forward_device(model, batch)
    ref, _ = emulated_backward(MAIN, w, batch, np.zeros((8, 1024, MAIN["d_in"])))
    assert rel_dev(ref, got) < BF16_TOL


def test_fully_masked_flags(fipa):
    """fully_masked (proj/src/flash_ipa.cpp:156-158): every row of a sample without a valid residue
    is flagged; partially masked or unmasked samples are not."""
    mask = np.ones((3, 70), dtype=bool)
    mask[1, :] = False
    mask[2, ::3] = False
    f = fipa.fully_masked(mask)
    assert f.shape == (3, 70) and f.dtype == bool
    assert f[1].all() and not f[0].any() and not f[2].any()
    assert not fipa.fully_masked(np.ones(5, bool)).any() and fipa.fully_masked(np.zeros(5, bool)).all()
