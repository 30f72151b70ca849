"""CPU: the C-ABI library and the drop-in Model surface, without GPU compute.

Covers: the library loads and exports every symbol include/fipa_b200.h declares; weights
init is bit-identical to the reference's IpaWeights::init; save/load is byte-identical to the
reference's weights file (proj/src/model_io.cpp:121-196) and rejects corrupted files the same
way; error types follow proj/python/bindings.cpp:176-178.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import fipa_oracle as fo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
HEADER = os.path.join(ROOT, "include", "fipa_b200.h")
TINY = dict(d_in=32, d_z=4, heads=2, c=8, n_query=2, n_value=2, rank=2)
MAIN = dict(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2)


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fipa_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(fipa):
    lib = ctypes.CDLL(fipa.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name


def test_c_abi_config_and_errors(fipa):
    lib = ctypes.CDLL(fipa.LIB_PATH)

    class Cfg(ctypes.Structure):
        _fields_ = [(n, ctypes.c_uint64) for n in ("d_in", "d_z", "heads", "c", "n_query", "n_value", "rank")] + [
            ("precision", ctypes.c_int32), ("enforce_head_cap", ctypes.c_int32)]

    lib.fipa_last_error.restype = ctypes.c_char_p
    lib.fipa_config_qk_width.restype = ctypes.c_uint64
    lib.fipa_config_v_width.restype = ctypes.c_uint64
    cfg = Cfg(**MAIN, precision=0, enforce_head_cap=1)
    assert lib.fipa_config_qk_width(ctypes.byref(cfg)) == 424
    assert lib.fipa_config_v_width(ctypes.byref(cfg)) == 420
    assert lib.fipa_config_validate(ctypes.byref(cfg)) == 1  # head cap -> FIPA_ERR_VALUE
    assert b"exceeds the cap of 256" in lib.fipa_last_error()
    cfg.enforce_head_cap = 0
    assert lib.fipa_config_validate(ctypes.byref(cfg)) == 0
    cfg.precision = 7
    assert lib.fipa_config_validate(ctypes.byref(cfg)) == 1
    handle = ctypes.c_void_p()
    cfg.precision = 0
    assert lib.fipa_layer_create(ctypes.byref(cfg), ctypes.byref(handle)) == 0
    lib.fipa_layer_workspace_size.restype = ctypes.c_size_t
    assert lib.fipa_layer_workspace_size(handle, ctypes.c_int64(2), ctypes.c_int64(100)) > 0
    # fused projection+pack (proj_pack.cu) -> attention -> output GEMM (+ recentre, cast)
    assert lib.fipa_layer_forward_launches(handle) == (6 if os.environ.get("FIPA_FUSED_PACK") == "0" else 4)
    lib.fipa_layer_destroy(handle)


@pytest.mark.parametrize("precision,tag", [("f64", "f64"), ("f32", "f32"), ("bf16", "f64")])
def test_model_init_weights_bit_identical_to_reference(fipa, precision, tag):
    """Model(seed) draws exactly IpaWeights::init(cfg, Rng(seed)) (proj/src/ipa.cpp:172-193);
    bf16 models keep float64 masters (rounded only on upload to the GPU)."""
    g = np.load(os.path.join(GOLD, "weights_seed7.npz"))
    w = fipa.Model(**TINY, precision=precision, seed=7).weights()
    for n in fo.WEIGHT_NAMES:
        assert np.array_equal(w[n], g[f"tiny/{tag}/{n}"]), n
    wm = fipa.Model(**MAIN, precision=precision, seed=7, enforce_head_cap=False).weights()
    for n in fo.WEIGHT_NAMES:
        assert np.array_equal(wm[n].ravel()[:64], g[f"main/{tag}/{n}/head"])
        assert np.sum(wm[n]) == float(g[f"main/{tag}/{n}/sum"])


@pytest.mark.parametrize("precision,fname", [("f64", "tiny_seed11.fipa"), ("f32", "tiny_f32_seed11.fipa")])
def test_save_is_byte_identical_and_load_round_trips(fipa, tmp_path, precision, fname):
    m = fipa.Model(**TINY, precision=precision, seed=11)
    path = str(tmp_path / "w.fipa")
    m.save(path)
    assert open(path, "rb").read() == open(os.path.join(GOLD, fname), "rb").read()
    other = fipa.Model(**TINY, precision=precision, seed=999)
    other.load(os.path.join(GOLD, fname))
    for n in fo.WEIGHT_NAMES:
        assert np.array_equal(other.weights()[n], m.weights()[n])


def test_corrupted_weights_files_are_rejected(fipa, tmp_path):
    """proj/tests/test_model_io.cpp:122-149."""
    good = open(os.path.join(GOLD, "tiny_seed11.fipa"), "rb").read()
    m = fipa.Model(**TINY)
    cases = {
        "missing": None,
        "magic": b"X" + good[1:],
        "version": good[:4] + bytes([99]) + good[5:],
        "truncated": good[: len(good) // 2],
        "trailing": good + b"\x00",
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.fipa"
        if data is not None:
            p.write_bytes(data)
        with pytest.raises(IOError):
            m.load(str(p))


def test_errors_surface_as_python_exceptions(fipa):
    """proj/tests/python/test_smoke.py:114-124 plus the GPU-only contract."""
    with pytest.raises(ValueError):
        fipa.Model(precision="f16")
    with pytest.raises(ValueError):
        fipa.Model(**MAIN)  # lifted width 424 > head cap (proj/src/ipa.cpp:16-20)
    m = fipa.Model(seed=12)
    p = fo.make_problem(fo.IpaConfig(), 12, seed=6)
    with pytest.raises(ValueError):
        m.flash(p.s, p.z1[:5], p.z2, p.rot, p.trans)
    with pytest.raises(ValueError):
        m.flash(p.s, p.z1, p.z2, p.rot, p.trans, mask=[True] * 3)
    with pytest.raises(ValueError):
        m.flash(p.s, p.z1, p.z2, p.rot[:, :2], p.trans)


def test_workspace_layout_is_consistent(fipa):
    m = fipa.Model(**MAIN, precision="bf16", enforce_head_cap=False)
    off, dims = m.workspace_layout(8, 1024)
    assert dims == [3744, 448, 448, 2432]
    present = [o for o in off if o >= 0]
    assert present == sorted(present) and all(o % 256 == 0 for o in present)
    assert m.workspace_size(8, 1024) > present[-1]
    mf = fipa.Model(**MAIN, precision="f32", enforce_head_cap=False)
    off32, _ = mf.workspace_layout(2, 64)
    assert off32[1] == -1  # no bf16 cast buffer on the fp32 path


def test_train_workspace_layout_slots(fipa):
    """Training layout: 11 slots; the fused backward's bf16 dQ / dK / dV copies (slots 8-10) exist
    at rank 2 and are absent (-1) for the materialised rank 3-4 backward, whose accumulator stride
    widens with the lifted rows."""
    m = fipa.Model(**MAIN, precision="bf16", enforce_head_cap=False)
    off, dims = m.train_workspace_layout(2, 512)
    assert len(off) == 11 and dims[0] == 448
    assert all(o >= 0 for o in off)
    assert len(set(off)) == 11 and all(o % 256 == 0 for o in off)
    assert m.train_workspace_size(2, 512) > max(off)
    m3 = fipa.Model(**dict(MAIN, rank=3), precision="bf16", enforce_head_cap=False)
    off3, dims3 = m3.train_workspace_layout(2, 512)
    assert off3[8:] == [-1, -1, -1] and dims3[0] >= 576
    # the materialised backward's [L, L] intermediates (12 bytes per head, query, key): quadratic in
    # L per sample group -- f(2L) - 2 f(L) = 2 * 12 H L^2 for the quadratic part
    excess = m3.train_workspace_size(1, 1024) - 2 * m3.train_workspace_size(1, 512)
    assert abs(excess - 2 * 12 * MAIN["heads"] * 512 ** 2) < 0.1 * 2 * 12 * MAIN["heads"] * 512 ** 2  # (- constant buffers)


def test_quadratic_arm_workspace_is_quadratic_and_flash_linear(fipa):
    """Memory model of the two arms (reference bench.cpp:151-155 estimate_reference_bytes and the
    paper's Fig. 2): the dense arm's workspace grows as (d_z + H) L^2, the flash workspace as L."""
    model = fipa.Model(**MAIN, precision="bf16", seed=0, enforce_head_cap=False)
    L0 = 8192
    d1, d2 = model.reference_workspace_size(1, L0), model.reference_workspace_size(1, 2 * L0)
    f1, f2 = model.workspace_size(1, L0), model.workspace_size(1, 2 * L0)
    assert 3.95 < d2 / d1 < 4.01
    assert 1.9 < f2 / f1 < 2.01
    quad = (MAIN["d_z"] + MAIN["heads"]) * (2 * L0) ** 2 * 4
    assert 0.95 < quad / d2 <= 1.0
