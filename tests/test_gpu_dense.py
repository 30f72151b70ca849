"""GPU: the quadratic-memory arm (Model.reference, dense.cu) and the generic attention entry points
(flash_attention / naive_attention) against the oracle, mirroring the reference pins:
  flash == quadratic          proj/tests/test_flash_ipa.cpp:170-202, tests/python/test_smoke.py:31-39
  kernel == naive             proj/tests/test_attention_kernel.cpp:100-136, 149-170, 315-336
  (ragged tiles, masks, +-700 logits, d = 300)
All fp32: gate 1e-4 (max|a-b| / max|ref|)."""

import numpy as np
import pytest

from helpers import F32_TOL, MAIN, TINY, make_batch, oracle_cfg, oracle_forward, oracle_weights_for, rel_dev
from oracle import fipa_oracle as fo

pytestmark = pytest.mark.gpu


def _oracle_reference(shape, w, batch):
    cfg = oracle_cfg(shape)
    return np.stack([fo.reference_forward(batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b],
                                          batch["trans"][b], batch["mask"][b], cfg, w)
                     for b in range(batch["s"].shape[0])])


@pytest.mark.parametrize("shape,B,L,mask_frac", [(TINY, 2, 37, 0.2), (MAIN, 1, 64, 0.1), (MAIN, 2, 130, 0.0),
                                                 (dict(MAIN, rank=3), 1, 48, 0.1)])
def test_reference_arm_matches_oracle(fipa, shape, B, L, mask_frac):
    model = fipa.Model(**shape, precision="f32", seed=5, enforce_head_cap=False)
    w = oracle_weights_for(model, "f32")
    batch = make_batch(shape, B, L, seed=300 + L, mask_frac=mask_frac)
    got = model.reference(batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"], mask=batch["mask"])
    ref = _oracle_reference(shape, w, batch)
    assert got.shape == ref.shape
    assert rel_dev(ref, got) < F32_TOL
    if mask_frac > 0:
        assert np.all(got[~batch["mask"].astype(bool)] == 0.0)


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_flash_equals_quadratic(fipa, precision):
    """Model.flash (linear memory) against Model.reference (quadratic) on the same inputs."""
    model = fipa.Model(**MAIN, precision=precision, seed=8, enforce_head_cap=False)
    batch = make_batch(MAIN, 1, 96, seed=17, mask_frac=0.1, bf16=precision == "bf16")
    args = (batch["s"], batch["z1"], batch["z2"], batch["rot"], batch["trans"])
    dense = model.reference(*args, mask=batch["mask"])
    flash = model.flash(*args, mask=batch["mask"])
    assert rel_dev(dense, flash) < (F32_TOL if precision == "f32" else 2e-2)
    w = oracle_weights_for(model, precision)
    assert rel_dev(oracle_forward(MAIN, w, batch), dense) < (F32_TOL if precision == "f32" else 2e-2)


def test_reference_arm_fully_masked_and_single_position(fipa):
    model = fipa.Model(**TINY, precision="f32", seed=2)
    batch = make_batch(TINY, 1, 9, seed=4)
    out = model.reference(batch["s"][0], batch["z1"][0], batch["z2"][0], batch["rot"][0], batch["trans"][0],
                          mask=[False] * 9)
    assert out.shape == (9, TINY["d_in"]) and np.all(out == 0.0)
    one = make_batch(TINY, 1, 1, seed=6)
    got = model.reference(one["s"][0], one["z1"][0], one["z2"][0], one["rot"][0], one["trans"][0])
    ref = _oracle_reference(TINY, oracle_weights_for(model, "f32"), one)[0]
    assert rel_dev(ref, got) < F32_TOL


def _qkv(rng, H, L, d, dv, scale=1.0):
    q = rng.standard_normal((H, L, d)) * scale
    k = rng.standard_normal((H, L, d))
    v = rng.standard_normal((H, L, dv))
    return q, k, v


@pytest.mark.parametrize("H,L,d,dv,scale,heads", [(1, 1, 8, 8, 1.0, False), (2, 37, 16, 24, 1.0, True),
                                                  (3, 130, 300, 70, 0.1, True), (1, 200, 64, 64, 40.0, False),
                                                  (2, 65, 33, 700, 1.0, True)])
@pytest.mark.parametrize("masked", [False, True])
def test_generic_attention(fipa, H, L, d, dv, scale, heads, masked):
    """flash_attention / naive_attention vs the oracle: ragged tiles, odd and wide d, key masks,
    logits of several hundred (scale 40 on d=64 puts rows at +-700, test_attention_kernel.cpp:149-170)."""
    rng = np.random.default_rng(L * 7 + d)
    q, k, v = _qkv(rng, H, L, d, dv, scale)
    mask = (rng.random(L) > 0.3) if masked else None
    if masked:
        mask[0] = True
    ref = fo.flash_attention(q, k, v, mask)
    if not heads:
        q, k, v, ref = q[0], k[0], v[0], ref[0]
    got_f = fipa.flash_attention(q, k, v, mask=mask)
    got_n = fipa.naive_attention(q, k, v, mask=mask)
    assert got_f.shape == ref.shape and got_n.shape == ref.shape
    tol = F32_TOL if scale < 10 else 1e-3  # +-700 logits: fp32 rounding of the logit itself
    assert rel_dev(ref, got_f) < tol
    assert rel_dev(ref, got_n) < tol


def test_generic_attention_all_keys_masked_and_errors(fipa):
    rng = np.random.default_rng(3)
    q, k, v = _qkv(rng, 2, 10, 4, 5)
    for fn in (fipa.flash_attention, fipa.naive_attention):
        out = fn(q, k, v, mask=[False] * 10)
        assert out.shape == (2, 10, 5) and np.all(out == 0.0)
        with pytest.raises(ValueError):
            fn(q, k[:, :9], v)
        with pytest.raises(ValueError):
            fn(q, k, v, mask=[True] * 3)
        with pytest.raises(ValueError):
            fn(q[0], k, v)
