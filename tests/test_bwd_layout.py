"""CPU: the device backward's layout bookkeeping (tests/bwd_emulation.py, a float64 emulation of
bwd_prep -> attention backward -> bwd_unpack in the lifted layout of pack.cu) reproduces the
reference-pinned oracle backward (oracle/fipa_oracle.flash_ipa_backward)."""

import numpy as np
import pytest

import bwd_emulation as be
from oracle import fipa_oracle as fo

CASES = [
    (dict(d_in=12, d_z=3, heads=2, c=4, n_query=2, n_value=3, rank=2), 9, 2.0, 0.2),
    (dict(d_in=32, d_z=8, heads=3, c=16, n_query=4, n_value=5, rank=3), 20, 20.0, 0.2),
    (dict(d_in=12, d_z=4, heads=1, c=5, n_query=1, n_value=1, rank=1), 6, 1.0, 0.0),
]


@pytest.mark.parametrize("shape,L,scale,mask_frac", CASES)
def test_emulated_device_backward_matches_oracle(shape, L, scale, mask_frac, monkeypatch):
    cfg = fo.IpaConfig(**shape, enforce_head_cap=False)
    w = fo.init_weights(cfg, 3)
    w["gamma_raw"] = np.linspace(-0.5, 0.8, cfg.heads)
    w["b_out"] = np.random.default_rng(2).standard_normal(cfg.d_in)
    p = fo.make_problem(cfg, L, 5, translation_scale=scale, mask_frac=mask_frac)
    dout = np.random.default_rng(0).standard_normal((L, cfg.d_in))
    ref = fo.flash_ipa_backward(p.s, p.z1, p.z2, p.rot, p.trans, p.mask, cfg, w, dout)
    monkeypatch.setattr(be, "EXACT_SPLIT", True)
    got, _ = be.backward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, p.mask, dout)
    for n in ref:
        assert fo.rel_dev(ref[n], got[n]) < 1e-8, n
    # with the bf16 hi/lo translation split the only loss is the dropped lo*lo product
    monkeypatch.setattr(be, "EXACT_SPLIT", False)
    got, _ = be.backward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, p.mask, dout)
    for n in ref:
        assert fo.rel_dev(ref[n], got[n]) < 2e-3, n


def test_large_L_checker_matches_oracle():
    """helpers.emulated_backward -- the checker the L >= 1024 GPU parity tests use (query-blocked,
    O(L) memory) -- against the dense oracle forward and backward at the north-star shape."""
    from helpers import MAIN, emulated_backward, make_batch, oracle_backward, oracle_forward

    cfg = fo.IpaConfig(**MAIN, enforce_head_cap=False)
    w = fo.init_weights(cfg, 1)
    w["gamma_raw"] = np.linspace(-0.6, 0.9, cfg.heads)
    batch = make_batch(MAIN, 2, 600, seed=3, mask_frac=0.1, bf16=True)  # > one 512-row block
    batch["mask"][1, :] = False  # a fully masked sample
    dout = np.random.default_rng(4).standard_normal((2, 600, cfg.d_in))
    out, g = emulated_backward(MAIN, w, batch, dout)
    assert fo.rel_dev(oracle_forward(MAIN, w, batch), out) < 1e-12
    ref = oracle_backward(MAIN, w, batch, dout)
    for n in ref:
        assert fo.rel_dev(ref[n], g[n]) < 1e-10, n
