"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front end over oracle/_ref/libfipa_ref.so -- the UNMODIFIED reference
library compiled from /root/reference/proj/src by oracle/Makefile, plus the
extern "C" shim in oracle/ref_shim.cpp.  Used to (a) generate the golden
fixtures under tests/golden/, (b) pin the numpy restatement, and (c) time the
reference CPU path in bench.py's cpu_baseline / --impl reference legs.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .fipa_oracle import WEIGHT_NAMES, IpaConfig, weight_shapes

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libfipa_ref.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = ctypes.c_char_p
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        raise {1: ValueError, 2: ArithmeticError, 3: IOError}.get(rc, RuntimeError)(msg)


def _dp(a):
    return a.ctypes.data_as(_D)


def _cfg(cfg: IpaConfig):
    return (ctypes.c_uint64 * 9)(*cfg.as_u64())


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _wptrs(cfg, w):
    arrs = [_c(w[n]) for n in WEIGHT_NAMES]
    ptrs = (_D * 10)(*[_dp(a) for a in arrs])
    scal = np.array([w.get("w_l", 0.0), w.get("w_c", 0.0)], dtype=np.float64)
    return arrs, ptrs, scal


def init_weights(cfg: IpaConfig, seed: int) -> dict:
    sh = weight_shapes(cfg)
    w = {n: np.zeros(sh[n]) for n in WEIGHT_NAMES}
    arrs, ptrs, scal = _wptrs(cfg, w)
    _check(lib().ref_init_weights(_cfg(cfg), ctypes.c_uint64(seed), ptrs, _dp(scal)))
    out = {n: a for n, a in zip(WEIGHT_NAMES, arrs)}
    out["w_l"], out["w_c"] = float(scal[0]), float(scal[1])
    return out


def _mask_ptr(mask, L):
    if mask is None:
        return None, None
    m = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8).reshape(L))
    return m, m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def flash_forward(cfg, w, s, z1, z2, rot, trans, mask=None, tile_rows=64, tile_cols=64, threads=1):
    L = s.shape[0]
    arrs, ptrs, scal = _wptrs(cfg, w)
    s, z1, z2, rot, trans = map(_c, (s, z1, z2, rot, trans))
    m, mp = _mask_ptr(mask, L)
    out = np.zeros((L, cfg.d_in))
    _check(lib().ref_flash_forward(_cfg(cfg), ptrs, _dp(scal), ctypes.c_uint64(L), _dp(s), _dp(z1),
                                   _dp(z2), _dp(rot), _dp(trans), mp, ctypes.c_uint64(tile_rows),
                                   ctypes.c_uint64(tile_cols), ctypes.c_int(threads), _dp(out)))
    return out


def reference_forward(cfg, w, s, z1, z2, rot, trans, mask=None):
    L = s.shape[0]
    arrs, ptrs, scal = _wptrs(cfg, w)
    s, z1, z2, rot, trans = map(_c, (s, z1, z2, rot, trans))
    m, mp = _mask_ptr(mask, L)
    out = np.zeros((L, cfg.d_in))
    _check(lib().ref_reference_forward(_cfg(cfg), ptrs, _dp(scal), ctypes.c_uint64(L), _dp(s),
                                       _dp(z1), _dp(z2), _dp(rot), _dp(trans), mp, _dp(out)))
    return out


def lift(cfg, w, s, z1, z2, rot, trans):
    L, H = s.shape[0], cfg.heads
    arrs, ptrs, scal = _wptrs(cfg, w)
    s, z1, z2, rot, trans = map(_c, (s, z1, z2, rot, trans))
    q = np.zeros((H, L, cfg.qk_width()))
    k = np.zeros((H, L, cfg.qk_width()))
    v = np.zeros((H, L, cfg.v_width()))
    _check(lib().ref_lift(_cfg(cfg), ptrs, _dp(scal), ctypes.c_uint64(L), _dp(s), _dp(z1), _dp(z2),
                          _dp(rot), _dp(trans), _dp(q), _dp(k), _dp(v)))
    return q, k, v


def flash_attention(q, k, v, mask=None, tile_rows=64, tile_cols=64, threads=1):
    q, k, v = map(_c, (q, k, v))
    H, L, dqk = q.shape
    dv = v.shape[2]
    m, mp = _mask_ptr(mask, L)
    out = np.zeros((H, L, dv))
    _check(lib().ref_flash_attention(ctypes.c_uint64(H), ctypes.c_uint64(L), ctypes.c_uint64(dqk),
                                     ctypes.c_uint64(dv), _dp(q), _dp(k), _dp(v), mp,
                                     ctypes.c_uint64(tile_rows), ctypes.c_uint64(tile_cols),
                                     ctypes.c_int(threads), _dp(out)))
    return out


def save_weights(cfg, w, path):
    arrs, ptrs, scal = _wptrs(cfg, w)
    _check(lib().ref_save_weights(_cfg(cfg), ptrs, _dp(scal), str(path).encode()))


def load_weights(cfg, path):
    sh = weight_shapes(cfg)
    w = {n: np.zeros(sh[n]) for n in WEIGHT_NAMES}
    arrs, ptrs, scal = _wptrs(cfg, w)
    _check(lib().ref_load_weights(_cfg(cfg), str(path).encode(), ptrs, _dp(scal)))
    out = {n: a for n, a in zip(WEIGHT_NAMES, arrs)}
    out["w_l"], out["w_c"] = float(scal[0]), float(scal[1])
    return out


def random_frames(seed, L, scale=1.0):
    rot = np.zeros((L, 3, 3))
    trans = np.zeros((L, 3))
    _check(lib().ref_random_frames(ctypes.c_uint64(seed), ctypes.c_uint64(L), ctypes.c_double(scale),
                                   _dp(rot), _dp(trans)))
    return rot, trans


def gaussian(seed, n, stddev=1.0):
    out = np.zeros(n)
    _check(lib().ref_gaussian(ctypes.c_uint64(seed), ctypes.c_uint64(n), ctypes.c_double(stddev), _dp(out)))
    return out


def knn_distogram(trans, k=20, n_bins=22, d_min=2.0, d_max=22.0, pe_dim=16):
    trans = _c(trans)
    L = trans.shape[0]
    out = np.zeros((L, k, n_bins + pe_dim))
    _check(lib().ref_knn_distogram(ctypes.c_uint64(L), _dp(trans), ctypes.c_uint64(k), ctypes.c_uint64(n_bins),
                                   ctypes.c_double(d_min), ctypes.c_double(d_max), ctypes.c_uint64(pe_dim), _dp(out)))
    return out


def build_factors(features, r, d_z, w1, w2):
    features, w1, w2 = map(_c, (features, w1, w2))
    L, f = features.shape
    z1 = np.zeros((L, r, d_z))
    z2 = np.zeros((L, r, d_z))
    _check(lib().ref_build_factors(ctypes.c_uint64(L), ctypes.c_uint64(f), _dp(features), ctypes.c_uint64(r),
                                   ctypes.c_uint64(d_z), _dp(w1), _dp(w2), _dp(z1), _dp(z2)))
    return z1, z2


# ------------------------------------------------------------ report / fit schema (f4)
def fit_polynomial(points):
    """bench.cpp:103-149 -> (a, b, r^2); NumericError -> ArithmeticError."""
    L = np.ascontiguousarray([p[0] for p in points], dtype=np.float64)
    y = np.ascontiguousarray([p[1] for p in points], dtype=np.float64)
    out = np.zeros(3)
    _check(lib().ref_fit_polynomial(ctypes.c_uint64(len(L)), _dp(L), _dp(y), _dp(out)))
    return float(out[0]), float(out[1]), float(out[2])


def _text(call):
    need = ctypes.c_uint64(0)
    _check(call(None, ctypes.c_uint64(0), ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value + 1)
    _check(call(buf, ctypes.c_uint64(need.value + 1), ctypes.byref(need)))
    return buf.value.decode()


def report_text(report, fmt):
    """report_to_csv / report_to_json (model_io.cpp:200-243) of a report.RunReport-shaped object."""
    U, P, Dp, Ip, S = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), _D, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p
    lib().ref_report_text.argtypes = [ctypes.c_int, S, S, U, S, P, P, Ip, P, Dp, U, S, S, Dp, U, S, Dp, Ip, U, S,
                                      ctypes.c_char_p, U, P]
    recs, fits, checks = report.records, report.fits, report.checks
    u64 = lambda xs: (ctypes.c_uint64 * max(1, len(xs)))(*xs)  # noqa: E731
    dbl = lambda xs: (ctypes.c_double * max(1, len(xs)))(*xs)  # noqa: E731
    i32 = lambda xs: (ctypes.c_int * max(1, len(xs)))(*xs)  # noqa: E731
    j = lambda xs: "\n".join(xs).encode()  # noqa: E731
    args = (ctypes.c_int(0 if fmt == "csv" else 1), report.command.encode(), report.config_echo.encode(),
            ctypes.c_uint64(len(recs)), j([r.arm for r in recs]), u64([r.length for r in recs]),
            u64([r.seed for r in recs]), i32([0 if r.precision == "f32" else 1 for r in recs]),
            u64([r.peak_bytes for r in recs]), dbl([r.seconds for r in recs]), ctypes.c_uint64(len(fits)),
            j([f.arm for f in fits]), j([f.metric for f in fits]),
            dbl([v for f in fits for v in (f.quadratic, f.linear, f.r_squared)]), ctypes.c_uint64(len(checks)),
            j([c.name for c in checks]), dbl([v for c in checks for v in (c.value, c.tolerance)]),
            i32([1 if c.passed else 0 for c in checks]), ctypes.c_uint64(len(report.notes)), j(report.notes))
    return _text(lambda b, cap, need: lib().ref_report_text(*args, b, cap, need))


def parse_records_csv_text(path):
    """parse_records_csv (model_io.cpp:260-306), returned re-serialised by report_to_csv."""
    return _text(lambda b, cap, need: lib().ref_parse_records_csv(str(path).encode(), b, cap, need))


def config_json(path=""):
    """config_to_json(load_config(path)) (model_io.cpp:308-405)."""
    return _text(lambda b, cap, need: lib().ref_config_json(str(path).encode(), b, cap, need))
