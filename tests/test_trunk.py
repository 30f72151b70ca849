"""BASELINE cfg3 trunk: layers + residual + per-layer backbone frame update.  The reference has no
trunk, so the oracle (fipa_oracle.trunk_forward) composes the reference's own
layer; the CPU tests pin that composition layer by layer to the compiled reference, and the GPU
tests compare fipa.Trunk (libfipa_b200.so) with the oracle."""

import numpy as np
import pytest

from helpers import MAIN, TINY, emulated_trunk, make_batch, rel_dev
from oracle import fipa_oracle as fo

SMALL = dict(d_in=16, d_z=4, heads=2, c=8, n_query=2, n_value=3, rank=2)


def _cfg(shape):
    return fo.IpaConfig(**shape, enforce_head_cap=False)


def test_trunk_oracle_layers_are_the_reference_layer():
    from oracle import ref

    if not ref.available():
        pytest.skip("compiled reference not available")
    cfg = _cfg(SMALL)
    layers, bbs = fo.init_trunk(cfg, 3, 4)
    p = fo.make_problem(cfg, 24, 8, translation_scale=3.0, mask_frac=0.2)
    s, rot, t = p.s, p.rot, p.trans
    for w, bb in zip(layers, bbs):
        s = s + ref.flash_forward(cfg, w, s, p.z1, p.z2, rot, t, p.mask)
        rot, t = fo.backbone_update(s, rot, t, p.mask, bb)
    got = fo.trunk_forward(p.s, p.z1, p.z2, p.rot, p.trans, p.mask, cfg, layers, bbs)
    assert rel_dev(s, got[0]) < 1e-12 and rel_dev(rot, got[1]) < 1e-12 and rel_dev(t, got[2]) < 1e-12
    # frames stay rotations; masked residues keep theirs
    assert np.abs(np.einsum("lab,lcb->lac", got[1], got[1]) - np.eye(3)).max() < 1e-12
    m = ~p.mask
    assert np.array_equal(got[1][m], p.rot[m]) and np.array_equal(got[2][m], p.trans[m])


def test_trunk_weights_bit_identical_to_oracle_init(fipa):
    cfg = _cfg(SMALL)
    trunk = fipa.Trunk(**SMALL, precision="bf16", seed=5, enforce_head_cap=False, n_layers=3)
    layers, bbs = fo.init_trunk(cfg, 3, 5)
    assert trunk.n_layers == 3
    for l in range(3):
        w, b = trunk.backbone(l)
        assert np.array_equal(w, bbs[l]["w"]) and np.array_equal(b, bbs[l]["b"])
        lw = trunk.layer(l).weights()
        assert all(np.array_equal(lw[n], layers[l][n]) for n in fo.WEIGHT_NAMES)
    trunk.set_backbone(1, np.ones((SMALL["d_in"], 6)), np.arange(6.0))
    assert np.array_equal(trunk.backbone(1)[1], np.arange(6.0))


def _gpu_trunk(trunk, batch):
    import torch

    dev = torch.device("cuda:0")
    B, L = batch["s"].shape[:2]
    t = {k: torch.from_numpy(np.ascontiguousarray(batch[k], dtype=np.float32)).to(dev)
         for k in ("s", "z1", "z2", "rot", "trans")}
    mask = torch.from_numpy(np.ascontiguousarray(batch["mask"], dtype=np.uint8)).to(dev)
    out = {k: torch.empty_like(t[k]) for k in ("s", "rot", "trans")}
    nbytes = trunk.workspace_size(B, L)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    trunk.forward_device(B, L, t["s"].data_ptr(), t["z1"].data_ptr(), t["z2"].data_ptr(), t["rot"].data_ptr(),
                         t["trans"].data_ptr(), mask.data_ptr(), out["s"].data_ptr(), out["rot"].data_ptr(),
                         out["trans"].data_ptr(), ws.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy().astype(np.float64) for k, v in out.items()}


def _trunk_weights(shape, trunk, precision):
    layers = []
    for l in range(trunk.n_layers):
        w = dict(trunk.layer(l).weights())
        if precision == "bf16":
            for n in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp", "w_out"):
                w[n] = fo.round_bf16(w[n])
        layers.append(w)
    bbs = [dict(zip(("w", "b"), trunk.backbone(l))) for l in range(trunk.n_layers)]
    return layers, bbs


def _oracle_trunk(shape, trunk, batch, precision, samples=None):
    """The oracle trunk (bf16: each layer reads its input s rounded to bf16, as the device's
    projection GEMM does; the fp32 residual stream and frame updates stay exact)."""
    cfg = _cfg(shape)
    layers, bbs = _trunk_weights(shape, trunk, precision)
    samples = range(batch["s"].shape[0]) if samples is None else samples
    if precision == "bf16":
        res = [emulated_trunk(cfg, layers, bbs, batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b],
                              batch["trans"][b], batch["mask"][b], layer_input=fo.round_bf16) for b in samples]
    else:
        res = [fo.trunk_forward(batch["s"][b], batch["z1"][b], batch["z2"][b], batch["rot"][b], batch["trans"][b],
                                batch["mask"][b], cfg, layers, bbs) for b in samples]
    return {k: np.stack([r[i] for r in res]) for i, k in enumerate(("s", "rot", "trans"))}


def test_emulated_trunk_is_the_oracle_trunk():
    """The large-L trunk checker (helpers.emulated_trunk: the lifted-row restatement, query-blocked)
    equals fipa_oracle.trunk_forward."""
    cfg = _cfg(MAIN)
    layers, bbs = fo.init_trunk(cfg, 2, 3)
    batch = make_batch(MAIN, 1, 200, seed=1, mask_frac=0.1, translation_scale=3.0)
    a = [batch[k][0] for k in ("s", "z1", "z2", "rot", "trans", "mask")]
    for x, y in zip(fo.trunk_forward(*a, cfg, layers, bbs), emulated_trunk(cfg, layers, bbs, *a)):
        assert rel_dev(x, y) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("f32", 1e-4), ("bf16", 2e-2)])
def test_trunk_matches_oracle(fipa, precision, tol):
    shape = MAIN
    trunk = fipa.Trunk(**shape, precision=precision, seed=9, enforce_head_cap=False, n_layers=3)
    batch = make_batch(shape, 2, 96, seed=90, mask_frac=0.1, bf16=precision == "bf16")
    got = _gpu_trunk(trunk, batch)
    ref = _oracle_trunk(shape, trunk, batch, precision)
    for k in ("s", "rot", "trans"):
        assert rel_dev(ref[k], got[k]) < tol, (k, rel_dev(ref[k], got[k]))


@pytest.mark.gpu
def test_trunk_cfg3_full_size(fipa):
    """BASELINE cfg3 as benched: 6 layers, B=4, L=2048, bf16, against the oracle trunk (checked on
    the first and last sample; gate 2e-2 on s, rot, trans)."""
    shape = MAIN
    trunk = fipa.Trunk(**shape, precision="bf16", seed=11, enforce_head_cap=False, n_layers=6)
    batch = make_batch(shape, 4, 2048, seed=91, mask_frac=0.05, bf16=True)
    got = _gpu_trunk(trunk, batch)
    ref = _oracle_trunk(shape, trunk, batch, "bf16", samples=(0, 3))
    for k in ("s", "rot", "trans"):
        g = got[k][[0, 3]]
        assert np.all(np.isfinite(got[k])), k
        assert rel_dev(ref[k], g) < 2e-2, (k, rel_dev(ref[k], g))


@pytest.mark.gpu
def test_trunk_six_layers_tiny(fipa):
    trunk = fipa.Trunk(**TINY, precision="f32", seed=2, enforce_head_cap=False, n_layers=6)
    batch = make_batch(TINY, 3, 40, seed=20, mask_frac=0.2)
    got = _gpu_trunk(trunk, batch)
    ref = _oracle_trunk(TINY, trunk, batch, "f32")
    for k in ("s", "rot", "trans"):
        assert rel_dev(ref[k], got[k]) < 1e-4, k
    m = ~batch["mask"].astype(bool)
    assert np.allclose(got["rot"][m], batch["rot"][m], atol=1e-6)
