"""GPU parity of the training path (forward_train + backward through the C ABI) against the
float64 oracle backward (oracle/fipa_oracle.flash_ipa_backward, pinned by finite differences of
the reference forward).  bf16 operands / fp32 accumulation: gate 2e-2 on max|a-b|/max|ref| per
gradient tensor, the oracle fed the same bf16-rounded inputs and weights."""

import numpy as np
import pytest

import bwd_emulation as be
from helpers import (BF16_TOL, MAIN, TINY, gpu_forward_device, gpu_train_device, make_batch,
                     oracle_backward, oracle_forward, oracle_weights_for, rel_dev, ws_view)
from oracle import fipa_oracle as fo

pytestmark = pytest.mark.gpu

GRADS = ("s", "z1", "z2", "rot", "trans") + fo.WEIGHT_NAMES
# gradients that reach their parameters only through the attention logits
LOGIT_PATH = ("rot", "w_q", "w_k", "w_qp", "w_kp", "gamma_raw")


def _model(fipa, shape, seed=0):
    m = fipa.Model(**shape, precision="bf16", seed=seed, enforce_head_cap=False)
    w = m.weights()
    # non-trivial gamma and output bias so their gradients are exercised
    w["gamma_raw"] = np.linspace(-0.6, 0.9, shape["heads"])
    w["b_out"] = np.random.default_rng(seed).standard_normal(shape["d_in"]) * 0.1
    m.set_weights(w)
    return m


def _check(fipa, shape, B, L, seed, mask_frac=0.0, scale=1.0, tol=BF16_TOL, tol_logit=None, bwd_ds=None,
           samples=None):
    model = _model(fipa, shape, seed)
    if bwd_ds is not None:
        model.set_tuning(bwd_ds=bwd_ds)
    w = oracle_weights_for(model, "bf16")
    batch = make_batch(shape, B, L, seed=seed, translation_scale=scale, mask_frac=mask_frac, bf16=True)
    dout = np.random.default_rng(seed + 1).standard_normal((B, L, shape["d_in"]))
    out, g, _, _ = gpu_train_device(model, batch, dout)
    ref_out = oracle_forward(shape, w, batch)
    assert rel_dev(ref_out, out) < tol
    ref = oracle_backward(shape, w, batch, dout)
    errs = {n: rel_dev(ref[n], g[n]) for n in GRADS}
    lim = {n: (tol_logit if tol_logit is not None and n in LOGIT_PATH else tol) for n in GRADS}
    bad = {n: e for n, e in errs.items() if not (np.isfinite(e) and e < lim[n])}
    assert not bad, f"gradients off: {bad} (all: {errs})"
    return errs


@pytest.mark.parametrize("L", [64, 200, 300])
def test_backward_main_shape(fipa, L):
    _check(fipa, MAIN, 2, L, seed=10 + L, mask_frac=0.1)


@pytest.mark.parametrize("ds", [0, 1])
def test_backward_both_dq_paths(fipa, ds):
    """dQ by the streaming attention kernel (bwd_ds=0) and by the batched GEMM over the
    dS the dK/dV kernel materialises (=1, the default for L <= 2048) -- each against the oracle."""
    _check(fipa, MAIN, 2, 257, seed=31, mask_frac=0.1, bwd_ds=ds)


def test_dq_paths_agree(fipa):
    """Same dS values either way (same formula, same bf16 rounding); the fp32 summation order of
    dQ differs, and the GEMM path hands dQ's scalar and pair columns to the unpack in bf16 while the
    streaming kernel keeps fp32 -- 2^-9-relative roundings, far inside the oracle gate."""
    model = _model(fipa, MAIN, 13)
    batch = make_batch(MAIN, 2, 320, seed=13, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(13).standard_normal((2, 320, MAIN["d_in"]))
    got = {}
    for ds in (0, 1):
        model.set_tuning(bwd_ds=ds)
        _, got[ds], _, _ = gpu_train_device(model, batch, dout)
    for n in GRADS:
        assert rel_dev(got[0][n], got[1][n]) < 4e-3, n


def test_micro_batched_capture_matches_one_chain(fipa):
    """micro=2 (two sample chunks on forked streams inside the captured graph, weight gradients
    accumulated by both chunks) against micro=1 and against the oracle: per-sample outputs are
    bitwise equal, the weight gradients differ only by fp32 summation order."""
    model = _model(fipa, MAIN, 17)
    B, L = 5, 192  # odd B: unequal chunks
    batch = make_batch(MAIN, B, L, seed=17, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(17).standard_normal((B, L, MAIN["d_in"]))
    res = {}
    for m in (1, 2):
        model.set_tuning(micro=m)
        assert model.tuning()["micro"] == m
        res[m] = gpu_train_device(model, batch, dout)[:2]
    assert np.array_equal(res[1][0], res[2][0])
    for n in GRADS:
        assert rel_dev(res[1][1][n], res[2][1][n]) < 1e-5, n
    w = oracle_weights_for(model, "bf16")
    ref = oracle_backward(MAIN, w, batch, dout)
    for n in GRADS:
        assert rel_dev(ref[n], res[2][1][n]) < BF16_TOL, n


@pytest.mark.parametrize("L", [200, 1024])
def test_backward_rank1(fipa, L):
    """z_factor_rank 1 (lifted widths 304 / 298: the fused kernels with narrower rows, prep's rank-1
    warp kernel, the general unpack form, rank-1 bf16 hand-off chunk masks) against the oracle."""
    _check(fipa, dict(MAIN, rank=1), 2, L, seed=60 + L, mask_frac=0.1)


def test_backward_sixteen_heads(fipa):
    """16 heads with narrower channels (the unpack's general form: more than 8 heads per residue,
    d(w_l w_bias) partials for 16 heads; the generic prep) against the oracle."""
    _check(fipa, dict(d_in=128, d_z=64, heads=16, c=64, n_query=4, n_value=8, rank=2), 2, 256, seed=71,
           mask_frac=0.1)


@pytest.mark.parametrize("rank,B,L", [(3, 2, 200), (4, 2, 320), (3, 1, 257)])
def test_backward_wide_lifted_rows(fipa, rank, B, L):
    """z_factor_rank 3-4 (lifted widths 576-704, wider than the fused attention backward holds):
    the materialised backward (batched tcgen05 GEMMs over the (sample, head) pairs) against the
    oracle at the same 2e-2 gate as every other training shape."""
    _check(fipa, dict(MAIN, rank=rank), B, L, seed=40 + rank + L, mask_frac=0.1)


def test_backward_wide_sample_groups(fipa):
    """The materialised backward in groups of one sample (a 1 MB intermediate budget forces
    att_samples = 1) gives the same gradients as one group of all samples."""
    shape = dict(MAIN, rank=3)
    model = _model(fipa, shape, 5)
    batch = make_batch(shape, 3, 192, seed=5, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(5).standard_normal((3, 192, shape["d_in"]))
    got = {}
    for cap in (2048, 1):
        model.set_tuning(ds_cap_mb=cap)
        got[cap] = gpu_train_device(model, batch, dout)[1]
    for n in GRADS:
        assert rel_dev(got[2048][n], got[1][n]) < 1e-5, n


def test_backward_tiny_shape(fipa):
    _check(fipa, TINY, 3, 37, seed=3, mask_frac=0.2)


def test_backward_protein_scale_coordinates(fipa):
    """Stress distribution: 30 A random translations (the reference's generator uses 1 A).
    Random frames that far apart make every query attend to ~one key (row-centred logits span
    ~3e4 log2 units), so the logit-path gradients are ill-conditioned in bf16: one-ulp changes of
    the lifted rows move them by a few percent (tools/diag_bwd.py: an exact float64 backward fed
    the device's own bf16 forward intermediates lands at the same error).  The value-path
    gradients keep the 2e-2 gate; the logit-path ones are held to 1e-1 (measured 2-7e-2)."""
    _check(fipa, MAIN, 1, 256, seed=4, scale=30.0, tol_logit=1e-1)


def test_backward_10A_coordinates(fipa):
    _check(fipa, MAIN, 1, 192, seed=5, scale=10.0, tol_logit=5e-2)


def test_backward_fully_masked_sample_is_zero(fipa):
    model = _model(fipa, MAIN, 2)
    batch = make_batch(MAIN, 2, 80, seed=2, bf16=True)
    batch["mask"][1, :] = False
    dout = np.random.default_rng(0).standard_normal((2, 80, MAIN["d_in"]))
    _, g, _, _ = gpu_train_device(model, batch, dout)
    for n in ("s", "z1", "z2", "rot", "trans"):
        assert np.all(g[n][1] == 0.0), n
        assert np.all(np.isfinite(g[n])), n


def test_training_forward_matches_inference_forward(fipa):
    model = _model(fipa, MAIN, 6)
    batch = make_batch(MAIN, 2, 130, seed=6, mask_frac=0.1, bf16=True)
    out_inf, _, _ = gpu_forward_device(model, batch)
    out_tr, _, _, _ = gpu_train_device(model, batch, np.zeros((2, 130, MAIN["d_in"])))
    assert np.array_equal(out_inf, out_tr)


@pytest.mark.parametrize("ds", [0, 1])
def test_attention_backward_stage_parity(fipa, ds):
    """dO_hat, D and the three attention accumulators against the layout emulation
    (tests/bwd_emulation.py) fed the device's own q/k/v_hat, O_hat and lse; dQ from both the
    streaming kernel and the materialised-dS GEMM."""
    B, L = 1, 160
    shape = MAIN
    model = _model(fipa, shape, 8)
    model.set_tuning(bwd_ds=ds)
    batch = make_batch(shape, B, L, seed=8, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(9).standard_normal((B, L, shape["d_in"]))
    _, _, ws, ((off, dims), (toff, tdims)) = gpu_train_device(model, batch, dout)
    n_proj, dqk_pad, dv_pad, nfeat = dims
    acc_ld = tdims[0]
    H = shape["heads"]
    q = ws_view(ws, off[3], H * L * dqk_pad, "bf16").reshape(H, L, dqk_pad)
    k = ws_view(ws, off[4], H * L * dqk_pad, "bf16").reshape(H, L, dqk_pad)
    v = ws_view(ws, off[5], H * L * dv_pad, "bf16").reshape(H, L, dv_pad)
    lse = ws_view(ws, off[7], H * L, "f32").reshape(H, L)
    o = ws_view(ws, toff[0], H * L * dv_pad, "f32").reshape(L, H, dv_pad).transpose(1, 0, 2)
    do = ws_view(ws, toff[1], H * L * dv_pad, "bf16").reshape(H, L, dv_pad)
    D = ws_view(ws, toff[2], H * L, "f32").reshape(H, L)
    o_ref, lse_ref = be.attention(q, k, v, L)
    assert rel_dev(o_ref, o) < 1e-2
    assert rel_dev(lse_ref, lse) < 1e-3
    assert rel_dev((do * o).sum(-1), D) < 1e-3
    dq_r, dk_r, dv_r = be.attention_backward(q, k, v, lse, do, D)
    # dQ in fp32; dK / dV: every column in the bf16 copies (slots 8, 9), the 32-column chunks with
    # point / translation columns also in fp32 (dK: [c, zq), dV: [c + r d_z, dv_used))
    c, zq, rdz = shape["c"], 176, shape["rank"] * shape["d_z"]
    geo = {"dk": (c, zq), "dv": (c + rdz, c + rdz + 6 + 3 * shape["n_value"])}
    # (dQ: the streaming kernel (ds = 0) writes fp32 whole; the materialised-dS GEMM a bf16 copy,
    # slot 10, plus the same fp32 geometry chunks as dK)
    geo["dq"] = geo["dk"]
    for name, idx, ref in (("dq", 3, dq_r), ("dk", 4, dk_r), ("dv", 5, dv_r)):
        got = ws_view(ws, toff[idx], H * L * acc_ld, "f32").reshape(L, H, acc_ld).transpose(1, 0, 2)
        if name == "dq" and ds == 0:
            assert rel_dev(ref[..., :432], got[..., :432]) < 1e-2, name
            continue
        slot16 = {"dq": 10, "dk": 8, "dv": 9}[name]
        g16 = ws_view(ws, toff[slot16], H * L * acc_ld, "bf16").reshape(L, H, acc_ld).transpose(1, 0, 2)
        assert rel_dev(ref[..., :432], g16[..., :432]) < 1e-2, name
        lo, hi = geo[name]
        lo32, hi32 = lo // 32 * 32, (hi + 31) // 32 * 32
        assert rel_dev(ref[..., lo32:hi32], got[..., lo32:hi32]) < 1e-2, name + " geometry chunks"


def test_flash_grad_host_api_matches_device(fipa):
    model = _model(fipa, TINY, 12)
    batch = make_batch(TINY, 2, 50, seed=12, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(1).standard_normal((2, 50, TINY["d_in"]))
    out_d, g_d, _, _ = gpu_train_device(model, batch, dout)
    out_h, g_h = model.flash_grad(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], dout,
                                  mask=batch["mask"])
    assert rel_dev(out_d, out_h) < 1e-6
    for n, m in (("s", "s"), ("z1", "z1"), ("rot", "rotations"), ("trans", "translations"), ("w_q", "w_q"),
                 ("gamma_raw", "gamma_raw"), ("w_out", "w_out")):
        assert rel_dev(g_d[n], g_h[m]) < 1e-5, n


def test_flash_grad_host_api_wide_rank(fipa):
    """The reference calling convention (float64 host arrays) over the materialised backward."""
    shape = dict(MAIN, rank=4)
    model = _model(fipa, shape, 14)
    batch = make_batch(shape, 2, 96, seed=14, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(2).standard_normal((2, 96, shape["d_in"]))
    out_d, g_d, _, _ = gpu_train_device(model, batch, dout)
    out_h, g_h = model.flash_grad(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], dout,
                                  mask=batch["mask"])
    assert rel_dev(out_d, out_h) < 1e-6
    for n, m in (("s", "s"), ("z2", "z2"), ("rot", "rotations"), ("w_k", "w_k"), ("w_bias", "w_bias")):
        assert rel_dev(g_d[n], g_h[m]) < 1e-5, n


def _check_large(fipa, B, L, seed, mask_frac, bwd_ds=None, oracle_samples=(), ds_cap_mb=None):
    """Large-L parity: forward output and all 15 gradients against the oracle-equivalent blocked
    emulation (helpers.emulated_backward: EXACT_SPLIT lifted restatement of the oracle backward,
    equal to it within 1e-14), plus the dense f64 oracle itself on `oracle_samples` (per-sample
    input gradients; weight gradients are batch sums and come from the emulation)."""
    from helpers import emulated_backward

    model = _model(fipa, MAIN, seed)
    if bwd_ds is not None:
        model.set_tuning(bwd_ds=bwd_ds)
    if ds_cap_mb is not None:
        model.set_tuning(ds_cap_mb=ds_cap_mb)
    w = oracle_weights_for(model, "bf16")
    batch = make_batch(MAIN, B, L, seed=seed, mask_frac=mask_frac, bf16=True)
    dout = np.random.default_rng(seed + 1).standard_normal((B, L, MAIN["d_in"]))
    out, g, _, _ = gpu_train_device(model, batch, dout)
    ref_out, ref = emulated_backward(MAIN, w, batch, dout)
    assert rel_dev(ref_out, out) < BF16_TOL
    errs = {n: rel_dev(ref[n], g[n]) for n in GRADS}
    bad = {n: e for n, e in errs.items() if not (np.isfinite(e) and e < BF16_TOL)}
    assert not bad, f"gradients off: {bad} (all: {errs})"
    for b in oracle_samples:
        one = {k: batch[k][b:b + 1] for k in batch}
        ro = oracle_backward(MAIN, w, one, dout[b:b + 1])
        for n in ("s", "z1", "z2", "rot", "trans"):
            assert rel_dev(ro[n][0], g[n][b]) < BF16_TOL, (b, n)
            assert rel_dev(ro[n][0], ref[n][b]) < 1e-10, (b, n)  # the emulation is the oracle
    return errs


def test_backward_bench_config(fipa):
    """Exactly the benched workload (bench.py default, BASELINE cfg2): B=8, L=1024, 10% masked
    residues, fwd+bwd through the materialised-dS path (its default at L <= 2048): ~7 waves of
    4-CTA clusters.  All 15 gradients; the dense oracle on samples 0 and 5."""
    _check_large(fipa, 8, 1024, seed=1234, mask_frac=0.1, oracle_samples=(0, 5))


@pytest.mark.parametrize("ds", [0, 1])
def test_backward_L2048(fipa, ds):
    """L = 2048 through the materialised-dS path and the streaming dQ kernel."""
    _check_large(fipa, 1, 2048, seed=2048, mask_frac=0.1, bwd_ds=ds)


@pytest.mark.parametrize("ds", [0, 1])
def test_backward_L4096(fipa, ds):
    """L = 4096: the materialised-dS path (the default up to L = 8192 / 2 GiB of dS) and the
    streaming dQ attention kernel (the path of every sharded training step)."""
    _check_large(fipa, 1, 4096, seed=4096, mask_frac=0.05, bwd_ds=ds)


@pytest.mark.parametrize("cap_mb", [8, 20])
def test_backward_query_chunked_ds(fipa, cap_mb):
    """Query-chunked materialised dS (the default beyond L = 8192 or 2 GiB, forced here with a small
    cap: 256- / 512-column chunks at B=2 L=1024): dK/dV accumulated over the chunks by TMA reduction,
    dQ one GEMM per chunk -- against the oracle-equivalent checker, and against the single-buffer
    path far inside the gate (fp32 summation order differs)."""
    errs = _check_large(fipa, 2, 1024, seed=77, mask_frac=0.1, ds_cap_mb=cap_mb)
    model = _model(fipa, MAIN, 77)
    batch = make_batch(MAIN, 2, 1024, seed=77, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(78).standard_normal((2, 1024, MAIN["d_in"]))
    _, g_full, _, _ = gpu_train_device(model, batch, dout)
    model.set_tuning(ds_cap_mb=cap_mb)
    assert model.tuning()["ds_cap_mb"] == cap_mb
    _, g_chunk, _, _ = gpu_train_device(model, batch, dout)
    for n in GRADS:
        # the single-buffer path hands dK / dV to the unpack as bf16 (scalar and pair columns), the
        # chunked one accumulates them in fp32 by TMA reduction: 2^-9-relative roundings (and fp32
        # summation order) apart, ~1e-3 on the gradients -- far inside the 2e-2 gate both pass above
        assert rel_dev(g_full[n], g_chunk[n]) < 4e-3, n
    assert errs


def test_host_paths_pipelined_and_float32(fipa):
    """The host entry points cut the batch into chunks (4 chunks here) pipelined over copy and compute
    streams; results equal the device path.  float32 arrays take the additive float32 path (float32
    out) with the same numbers."""
    model = _model(fipa, MAIN, 14)
    B, L = 8, 256
    batch = make_batch(MAIN, B, L, seed=14, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(2).standard_normal((B, L, MAIN["d_in"]))
    out_d, g_d, _, _ = gpu_train_device(model, batch, dout)
    args = [batch[k] for k in ("s", "z1", "z2", "rot", "trans")]
    out_h = model.flash(*args, mask=batch["mask"])
    assert out_h.dtype == np.float64 and rel_dev(out_d, out_h) < 1e-6
    out_g, g_h = model.flash_grad(*args, dout, mask=batch["mask"])
    assert rel_dev(out_d, out_g) < 1e-6
    for n, m in (("s", "s"), ("z2", "z2"), ("rot", "rotations"), ("trans", "translations"), ("w_k", "w_k"),
                 ("w_bias", "w_bias"), ("w_out", "w_out"), ("b_out", "b_out")):
        assert rel_dev(g_d[n], g_h[m]) < 1e-5, n
    a32 = [a.astype(np.float32) for a in args]
    out_32 = model.flash(*a32, mask=batch["mask"])
    assert out_32.dtype == np.float32 and rel_dev(out_h, out_32) < 1e-6
    o32, g32 = model.flash_grad(*a32, dout.astype(np.float32), mask=batch["mask"])
    assert o32.dtype == np.float32 and g32["s"].dtype == np.float32
    assert rel_dev(g_h["s"], g32["s"]) < 1e-5 and rel_dev(g_h["w_q"], g32["w_q"]) < 1e-5
