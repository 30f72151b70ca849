"""CPU: the report / configuration schema (paper_2505_11580_b200/report.py) against the reference's
own expectations (proj/tests/test_model_io.cpp:151-298, proj/tests/test_bench.cpp:46-83)."""

import json

import numpy as np
import pytest

from paper_2505_11580_b200 import report as rp


def _sample_report():
    r = rp.RunReport(command="scaling", config_echo=rp.config_to_json(rp.load_config("")))
    r.records = [rp.RunRecord("reference", 128, 7, "f64", 123456, 0.125),
                 rp.RunRecord("flash", 256, 7, "f32", 654321, 1.0 / 3.0)]
    r.fits = [rp.FitSummary("flash", "peak_bytes", 1e-3, 2.5, 0.999)]
    r.checks = [rp.CheckOutcome("scaling/flash/quadratic-share", 0.001, 0.01, True)]
    r.notes = ["reference arm skipped at L=8192: estimated peak exceeds budget"]
    return r


def test_records_csv_pinned_order_and_exact_round_trip(tmp_path):
    rep = _sample_report()
    csv = rp.report_to_csv(rep)
    assert csv.startswith("arm,L,seed,precision,peak_bytes,seconds\n")
    p = tmp_path / "records.csv"
    p.write_text(csv)
    back = rp.parse_records_csv(str(p))
    assert back == rep.records  # seconds survive the 17-digit text form bit-exactly


def test_header_only_csv_and_malformed_inputs(tmp_path):
    p = tmp_path / "r.csv"
    p.write_text(rp.CSV_HEADER + "\n")
    assert rp.parse_records_csv(str(p)) == []
    with pytest.raises(IOError):
        rp.parse_records_csv(str(tmp_path / "missing.csv"))
    for body in ("arm,length,seed,precision,peak_bytes,seconds\n",
                 rp.CSV_HEADER + "\nflash,128,7,f64\n",
                 rp.CSV_HEADER + "\nflash,huge,7,f64,1,0.5\n"):
        p.write_text(body)
        with pytest.raises(IOError):
            rp.parse_records_csv(str(p))


def test_json_report_carries_records_fits_checks_notes(tmp_path):
    rep = _sample_report()
    doc = json.loads(rp.report_to_json(rep))
    assert doc["command"] == "scaling"
    assert len(doc["records"]) == 2 and doc["records"][0]["arm"] == "reference" and doc["records"][0]["L"] == 128
    assert doc["records"][1]["precision"] == "f32"
    assert doc["fits"][0]["metric"] == "peak_bytes"
    assert doc["checks"][0]["pass"] is True
    assert "8192" in doc["notes"][0]
    assert doc["config"]["model"]["d_in"] == 32
    rp.emit_report(rep, "csv", str(tmp_path / "e.csv"))
    rp.emit_report(rep, "json", str(tmp_path / "e.json"))
    assert len(rp.parse_records_csv(str(tmp_path / "e.csv"))) == 2
    assert len(json.loads((tmp_path / "e.json").read_text())["records"]) == 2
    with pytest.raises(ValueError):
        rp.emit_report(rep, "yaml", str(tmp_path / "e.yaml"))


def test_default_config_and_overrides(tmp_path):
    cfg = rp.load_config("")
    assert (cfg.model.d_in, cfg.model.heads, cfg.model.precision) == (32, 2, "f64")
    assert (cfg.distogram.k, cfg.distogram.n_bins) == (20, 22)
    assert cfg.lengths == [] and cfg.arms == ["reference", "flash"] and cfg.trials == 100
    assert cfg.tile_rows == 64 and cfg.reference_byte_budget == 1500000000 and cfg.threads == 1
    cfg.validate()
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"model": {"heads": 4, "precision": "f32", "rank": 3}, "distogram": {"k": 10},
                             "bench": {"lengths": [32, 64], "arms": ["flash"], "trials": 5, "tile_rows": 16,
                                       "tile_cols": 32, "threads": 2, "translation_scale": 2.5,
                                       "reference_byte_budget": 1000}}))
    c = rp.load_config(str(p))
    assert (c.model.heads, c.model.precision, c.model.rank, c.model.d_in) == (4, "f32", 3, 32)
    assert (c.distogram.k, c.distogram.n_bins) == (10, 22)
    assert c.lengths == [32, 64] and c.arms == ["flash"] and c.trials == 5
    assert (c.tile_rows, c.tile_cols, c.threads, c.translation_scale, c.reference_byte_budget) == (16, 32, 2, 2.5, 1000)
    echo = rp.config_to_json(c)
    p.write_text(echo)
    back = rp.load_config(str(p))
    assert back == c


def test_broken_configs_rejected(tmp_path):
    p = tmp_path / "bad.json"
    with pytest.raises(IOError):
        rp.load_config(str(p))
    p.write_text("{not json")
    with pytest.raises(IOError):
        rp.load_config(str(p))
    p.write_text(json.dumps({"model": {"precision": "f16"}}))
    with pytest.raises(ValueError):
        rp.load_config(str(p))
    p.write_text(json.dumps({"bench": {"arms": ["turbo"]}}))
    with pytest.raises(ValueError):
        rp.load_config(str(p)).validate()


def test_fit_polynomial_matches_reference_cases():
    a, b, r2 = rp.fit_polynomial([(L, 3.0 * L) for L in (64.0, 128.0, 256.0, 512.0)])
    assert abs(a) < 1e-9 and b == pytest.approx(3.0, rel=1e-9) and r2 == pytest.approx(1.0, abs=1e-12)
    a, b, r2 = rp.fit_polynomial([(L, 2.0 * L * L + L) for L in (100.0, 300.0, 1000.0, 4000.0, 8192.0)])
    assert a == pytest.approx(2.0, rel=1e-9) and b == pytest.approx(1.0, rel=1e-6) and r2 == pytest.approx(1.0)
    rng = np.random.default_rng(120)
    pts = [(L, (5.0 * L * L + 400.0 * L) * (1 + 0.01 * rng.standard_normal())) for L in
           (128.0, 256.0, 512.0, 1024.0, 2048.0, 4096.0)]
    a, b, r2 = rp.fit_polynomial(pts)
    assert a == pytest.approx(5.0, rel=0.15) and r2 > 0.99
    for bad in ([], [(64.0, 1.0)], [(64.0, 1.0), (64.0, 2.0), (64.0, 3.0)]):
        with pytest.raises(ArithmeticError):
            rp.fit_polynomial(bad)


def test_fit_command_and_scaling_checks(tmp_path):
    rep = rp.RunReport(command="scaling")
    for L in (1024, 2048, 4096):
        rep.records.append(rp.RunRecord("flash", L, 0, "bf16", 1000 * L, 1e-6 * L))
        rep.records.append(rp.RunRecord("reference", L, 0, "f32", 136 * 4 * L * L + 5000 * L, 1e-9 * L * L))
    rp.scaling_checks(rep, "flash")
    rp.scaling_checks(rep, "reference")
    assert rep.all_pass(), rep.checks
    names = [c.name for c in rep.checks]
    assert names == ["scaling/flash/quadratic-share", "scaling/flash/memory-fit-r2",
                     "scaling/reference/quadratic-share@L=2048"]
    p = tmp_path / "r.csv"
    rp.emit_report(rep, "csv", str(p))
    fit = rp.run_fit(str(p), "peak_bytes")
    assert [f.arm for f in fit.fits] == ["flash", "reference"]
    assert fit.fits[1].quadratic == pytest.approx(544.0, rel=1e-9)


# ------------------------------------------------------------------ pinned to the compiled reference
def _ref():
    from oracle import ref

    if not ref.available():
        pytest.skip("compiled reference not available (make -C oracle)")
    return ref


def _rich_report():
    r = rp.RunReport(command="scaling", config_echo=rp.config_to_json(rp.load_config("")))
    vals = [0.125, 1.0 / 3.0, 1e-9, 12345.678901234567, 2.0 ** -40, 7.0, 0.1 + 0.2]
    r.records = [rp.RunRecord("flash" if i % 2 else "reference", 128 << i, 7 + i, "f32" if i % 3 else "f64",
                              10 ** i + 3, v) for i, v in enumerate(vals)]
    r.fits = [rp.FitSummary("flash", "peak_bytes", 1e-3, 2.5, 0.999),
              rp.FitSummary("reference", "seconds", 3.25e-9, -1.5e-7, 1.0 / 7.0)]
    r.checks = [rp.CheckOutcome("scaling/flash/quadratic-share", 0.001, 0.01, True),
                rp.CheckOutcome("scaling/reference/r2", 0.5, 0.99, False)]
    r.notes = ["reference arm skipped at L=8192: estimated peak exceeds budget", "second note"]
    return r


def test_report_text_byte_identical_to_reference():
    """report_to_csv / report_to_json text equals the reference's (proj/src/model_io.cpp:200-243)
    byte for byte: 17-digit CSV seconds, nlohmann's sorted keys and number forms."""
    ref = _ref()
    rep = _rich_report()
    assert rp.report_to_csv(rep) == ref.report_text(rep, "csv")
    assert rp.report_to_json(rep) == ref.report_text(rep, "json")


def test_records_csv_parsed_identically(tmp_path):
    """Our CSV parsed by the reference (model_io.cpp:260-306) and re-emitted is the same text; the
    reference's CSV parsed by ours gives the same records."""
    ref = _ref()
    rep = _rich_report()
    p = tmp_path / "r.csv"
    p.write_text(rp.report_to_csv(rep))
    assert ref.parse_records_csv_text(p) == rp.report_to_csv(rep)
    p.write_text(ref.report_text(rep, "csv"))
    assert rp.parse_records_csv(str(p)) == rep.records
    for body in ("arm,length,seed,precision,peak_bytes,seconds\n", rp.CSV_HEADER + "\nflash,128,7,f64\n"):
        p.write_text(body)
        with pytest.raises(IOError):
            ref.parse_records_csv_text(p)
        with pytest.raises(IOError):
            rp.parse_records_csv(str(p))


@pytest.mark.parametrize("seed", range(6))
def test_fit_polynomial_matches_reference(seed):
    """fit_polynomial (proj/src/bench.cpp:103-149) on random designs, noisy and exact."""
    ref = _ref()
    rng = np.random.default_rng(seed)
    Ls = np.sort(rng.choice([128, 256, 512, 1024, 2048, 4096, 8192, 16384], size=4 + seed % 4, replace=False))
    a, b = rng.uniform(1e-6, 1e-2), rng.uniform(-1.0, 5.0)
    ys = a * Ls ** 2 + b * Ls
    if seed % 2:
        ys = ys * (1 + 0.05 * rng.standard_normal(len(Ls)))
    pts = list(zip(Ls.astype(float), ys))
    want = ref.fit_polynomial(pts)
    got = rp.fit_polynomial(pts)
    for w_, g_ in zip(want, got):
        assert abs(w_ - g_) <= 1e-12 * max(1.0, abs(w_))


def test_fit_polynomial_degenerate_designs_match_reference():
    ref = _ref()
    for pts in ([(128.0, 1.0)], [(256.0, 1.0), (256.0, 2.0)], [(0.0, 1.0), (0.0, 3.0)]):
        with pytest.raises(ArithmeticError):
            ref.fit_polynomial(pts)
        with pytest.raises(ArithmeticError):
            rp.fit_polynomial(pts)


def test_config_json_matches_reference(tmp_path):
    """load_config + config_to_json (model_io.cpp:308-405): defaults and a partial file."""
    ref = _ref()
    assert rp.config_to_json(rp.load_config("")) == ref.config_json("")
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"model": {"d_in": 64, "heads": 4, "precision": "f32"},
                             "distogram": {"k": 12}, "bench": {"lengths": [128, 256], "trials": 3}}))
    assert rp.config_to_json(rp.load_config(str(p))) == ref.config_json(str(p))
