"""Pair-factor producer: knn_distogram / positional_encoding / build_factors
(proj/src/pair_features.cpp:10-97).  The numpy restatement is pinned to the compiled reference;
the GPU kernels must reproduce the reference's neighbour choice exactly (integer work: indices and
bins bit-exact, the sinusoids to float32 rounding).  Cases follow the reference's own tests
(proj/tests/test_pair_features.cpp:65-136): nearest selection with lower-index tie-break, clipping
into the end bins, invariance under rigid motion, input validation."""

import numpy as np
import pytest

from oracle import fipa_oracle as fo


def _line(n):
    """Points on a line with duplicated positions -> exact distance ties."""
    x = np.array([0.0, 1.0, 1.0, 2.5, 2.5, 2.5, 6.0, 9.0, 14.0, 30.0][:n])
    return np.stack([x, np.zeros(n), np.zeros(n)], 1)


def _cloud(n, seed, scale=6.0):
    """A float64 point cloud (NOT rounded to float32: the f64 API must keep every bit)."""
    return np.random.default_rng(seed).standard_normal((n, 3)) * scale


def _near_ties(n, seed):
    """Shells of points whose distances to their centre differ by ~1e-12 A: they tie after a
    float32 rounding, and the higher index is always the nearer one, so a rounded path picks the
    wrong neighbour (lower-index tie-break) while the f64 reference does not."""
    rng = np.random.default_rng(seed)
    pts = [rng.standard_normal(3) * 8.0 for _ in range(n // 8)]
    out = []
    for c in pts:
        out.append(c)
        for m in range(7):
            u = rng.standard_normal(3)
            u /= np.linalg.norm(u)
            out.append(c + u * (3.0 - 1e-12 * m))  # later points slightly closer
    return np.asarray(out[:n])


def test_oracle_matches_reference_knn_and_factors():
    from oracle import ref

    if not ref.available():
        pytest.skip("compiled reference not available")
    for pts, kw in ((_line(10), dict(k=4, n_bins=5, d_min=0.5, d_max=5.0, pe_dim=4)),
                    (_cloud(80, 1), dict(k=20)), (_cloud(40, 2, 30.0), dict(k=7, n_bins=8, pe_dim=6))):
        assert np.array_equal(ref.knn_distogram(pts, **kw), fo.knn_distogram(pts, **kw))
    rng = np.random.default_rng(0)
    f = rng.standard_normal((30, 12))
    w1, w2 = rng.standard_normal((12, 6)), rng.standard_normal((12, 6))
    z = ref.build_factors(f, 2, 3, w1, w2)
    zz = fo.build_factors(f, 2, 3, w1, w2)
    assert np.abs(z[0] - zz[0]).max() < 1e-12 and np.abs(z[1] - zz[1]).max() < 1e-12


def test_oracle_tie_break_clipping_and_invariance():
    feats = fo.knn_distogram(_line(10), k=3, n_bins=5, d_min=0.5, d_max=5.0, pe_dim=4)
    # residue 1 (x=1): nearest is residue 2 (same position, distance 0) then 0 (d=1); bins clip to 0
    assert feats[1, 0, 0] == 1.0 and feats[1, 1, 0] == 1.0
    # residue 3's tie between 4 and 5 (both distance 0) goes to the lower index first
    np.testing.assert_allclose(feats[3, 0, 5:], fo.positional_encoding([1], 4)[0])
    np.testing.assert_allclose(feats[3, 1, 5:], fo.positional_encoding([2], 4)[0])
    far = fo.knn_distogram(_line(10), k=1, n_bins=5, d_min=0.5, d_max=5.0, pe_dim=4)
    assert far[9, 0, 4] == 1.0  # 16 A away -> clipped into the last bin
    pts = _cloud(50, 3)
    rot, t = fo.random_rototranslation(fo.Rng(4), 10.0)
    moved = pts @ rot.T + t
    assert np.abs(fo.knn_distogram(pts) - fo.knn_distogram(moved)).max() < 1e-9


def test_input_validation_matches_reference(fipa):
    pts = _cloud(10, 5)
    for kw in (dict(k=0), dict(k=10), dict(n_bins=1), dict(d_min=5.0, d_max=5.0), dict(pe_dim=3)):
        with pytest.raises(ValueError):
            fipa.knn_distogram(pts, **{**dict(k=4), **kw})
        with pytest.raises(ValueError):
            fo.knn_distogram(pts, **{**dict(k=4), **kw})
    with pytest.raises(ValueError):
        fipa.knn_distogram(pts[:1], k=1)


def _check_feats(ref, got, n_bins):
    assert np.array_equal(ref[..., :n_bins], got[..., :n_bins])  # neighbour choice + bins: exact
    # sinusoids: float64 on both sides (device sincos vs glibc: a few ulp); wrong neighbours would
    # show as O(1) differences of the offset encoding
    assert np.abs(ref[..., n_bins:] - got[..., n_bins:]).max() < 1e-12


def test_near_tie_cloud_separates_f32_from_f64():
    """The near-tie fixture really is a float32/float64 discriminator for the oracle."""
    pts = _near_ties(64, 3)
    exact = fo.knn_distogram(pts, k=6)
    rounded = fo.knn_distogram(pts.astype(np.float32).astype(np.float64), k=6)
    assert not np.array_equal(exact[..., 22:], rounded[..., 22:])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_gpu_knn_near_ties_bit_exact_vs_compiled_reference(fipa, seed):
    """f64 clouds with engineered near-ties (distances 1e-12 apart): the GPU's neighbour indices and
    bins equal the compiled reference's (oracle/_ref, proj/src/pair_features.cpp:29-45) bit for bit."""
    from oracle import ref

    pts = _near_ties(256, seed)
    kw = dict(k=7, n_bins=16, d_min=2.0, d_max=4.0, pe_dim=8)
    got = fipa.knn_distogram(pts, **kw)
    want = ref.knn_distogram(pts, **kw) if ref.available() else fo.knn_distogram(pts, **kw)
    _check_feats(want, got, kw["n_bins"])
    got_b = fipa.knn_distogram(np.stack([pts, pts[::-1].copy()]), **kw)  # batched path, same rule
    _check_feats(want, got_b[0], kw["n_bins"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["line", "cloud", "far", "batched"])
def test_gpu_knn_distogram_matches_oracle(fipa, case):
    if case == "line":
        pts, kw = _line(10), dict(k=6, n_bins=5, d_min=0.5, d_max=5.0, pe_dim=4)
    elif case == "cloud":
        pts, kw = _cloud(700, 6), dict()
    elif case == "far":
        pts, kw = _cloud(300, 7, 40.0), dict(k=33, n_bins=10, pe_dim=8)
    else:
        pts = np.stack([_cloud(130, 8), _cloud(130, 9)])
        kw = dict(k=12)
    got = fipa.knn_distogram(pts, **kw)
    ref = np.stack([fo.knn_distogram(p, **kw) for p in pts]) if pts.ndim == 3 else fo.knn_distogram(pts, **kw)
    _check_feats(ref, got, kw.get("n_bins", 22))


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("bf16", 2e-2), ("f32", 1e-5)])
def test_gpu_build_factors(fipa, precision, tol):
    rng = np.random.default_rng(1)
    L, k, f0, r, dz = 200, 20, 38, 2, 128
    feats = fo.knn_distogram(_cloud(L, 10), k=k).reshape(L, k * f0)
    w1 = rng.standard_normal((k * f0, r * dz)) / np.sqrt(k * f0)
    w2 = rng.standard_normal((k * f0, r * dz)) / np.sqrt(k * f0)
    z1, z2 = fipa.build_factors(feats, r, dz, w1, w2, precision=precision)
    if precision == "bf16":
        feats, w1, w2 = fo.round_bf16(feats), fo.round_bf16(w1), fo.round_bf16(w2)
    e1, e2 = fo.build_factors(feats, r, dz, w1, w2)
    assert fo.rel_dev(e1, z1) < tol and fo.rel_dev(e2, z2) < tol
