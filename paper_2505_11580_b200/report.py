"""Benchmark report and configuration schema of the reference, so GPU
measurements can be diffed against CPU records and refit with the reference's `fipa fit` semantics.

Mirrors proj/include/fipa/model_io.hpp:28-105 and proj/src/model_io.cpp:198-405:
  RunRecord / FitSummary / CheckOutcome / RunReport      model_io.hpp:30-75
  report_to_csv / report_to_json / emit_report           model_io.cpp:200-258
  parse_records_csv                                      model_io.cpp:260-306
  BenchConfig / load_config / config_to_json / validate  model_io.cpp:308-405
  fit_polynomial (y = a L^2 + b L, normalised design)    proj/src/bench.cpp:103-149
Same CSV header and JSON keys, same error types (ValueError for bad arguments / degenerate
designs reported as ArithmeticError like the reference's NumericError, IOError for files).
Precision names accept "bf16" in addition to the reference's "f32" / "f64".
"""

from __future__ import annotations

import dataclasses
import json
import math
import sys
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

CSV_HEADER = "arm,L,seed,precision,peak_bytes,seconds"
PRECISIONS = ("f32", "f64", "bf16")
ARMS = ("reference", "flash")


@dataclass
class RunRecord:
    arm: str
    length: int
    seed: int
    precision: str
    peak_bytes: int
    seconds: float


@dataclass
class FitSummary:
    arm: str
    metric: str  # "peak_bytes" or "seconds"
    quadratic: float
    linear: float
    r_squared: float


@dataclass
class CheckOutcome:
    name: str
    value: float
    tolerance: float
    passed: bool


@dataclass
class RunReport:
    command: str = ""
    config_echo: str = ""
    records: List[RunRecord] = field(default_factory=list)
    fits: List[FitSummary] = field(default_factory=list)
    checks: List[CheckOutcome] = field(default_factory=list)
    notes: List[str] = field(default_factory=list)

    def all_pass(self) -> bool:
        return all(c.passed for c in self.checks)


def _repr_g17(x: float) -> str:
    # std::ostream with precision(17): general format, 17 significant digits
    return format(x, ".17g")


def report_to_csv(report: RunReport) -> str:
    lines = [CSV_HEADER]
    for r in report.records:
        lines.append(f"{r.arm},{r.length},{r.seed},{r.precision},{r.peak_bytes},{_repr_g17(r.seconds)}")
    return "\n".join(lines) + "\n"


def report_to_json(report: RunReport) -> str:
    j = {
        "command": report.command,
        "config": json.loads(report.config_echo) if report.config_echo else {},
        "records": [{"arm": r.arm, "L": r.length, "seed": r.seed, "precision": r.precision,
                     "peak_bytes": r.peak_bytes, "seconds": r.seconds} for r in report.records],
        "fits": [{"arm": f.arm, "metric": f.metric, "quadratic": f.quadratic, "linear": f.linear,
                  "r_squared": f.r_squared} for f in report.fits],
        "checks": [{"name": c.name, "value": c.value, "tolerance": c.tolerance, "pass": c.passed}
                   for c in report.checks],
        "notes": list(report.notes),
    }
    return json.dumps(j, indent=2, sort_keys=True) + "\n"  # nlohmann::json: keys sorted, dump(2)


def emit_report(report: RunReport, fmt: str, path: str = "-") -> None:
    if fmt == "csv":
        text = report_to_csv(report)
    elif fmt == "json":
        text = report_to_json(report)
    else:
        raise ValueError(f"unknown report format '{fmt}' (expected csv or json)")
    if not path or path == "-":
        sys.stdout.write(text)
        return
    try:
        with open(path, "w", newline="") as f:
            f.write(text)
    except OSError as exc:
        raise IOError(f"cannot open '{path}' for writing") from exc


def parse_records_csv(path: str) -> List[RunRecord]:
    try:
        with open(path, newline="") as f:
            lines = f.read().splitlines()
    except OSError as exc:
        raise IOError(f"cannot open '{path}' for reading") from exc
    if not lines:
        raise IOError("records csv: empty file")
    if lines[0] != CSV_HEADER:
        raise IOError(f"records csv: unexpected header '{lines[0]}'")
    out = []
    for n, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        cells = line.split(",")
        if len(cells) != 6:
            raise IOError(f"records csv: line {n} has {len(cells)} fields, expected 6")
        if cells[3] not in PRECISIONS:
            raise ValueError(f"unknown precision '{cells[3]}'")
        try:
            out.append(RunRecord(cells[0], int(cells[1]), int(cells[2]), cells[3], int(cells[4]), float(cells[5])))
        except ValueError as exc:
            raise IOError(f"records csv: line {n} is not numeric") from exc
    return out


def fit_polynomial(points: Sequence[Tuple[float, float]]) -> Tuple[float, float, float]:
    """Least squares y = a L^2 + b L on u = L / L_max (bench.cpp:103-149) -> (a, b, r^2)."""
    if len(points) < 2 or len({p[0] for p in points}) < 2:
        raise ArithmeticError("degenerate design: fitting quadratic+linear terms needs at least two distinct lengths")
    l_max = max(abs(p[0]) for p in points)
    if l_max <= 0:
        raise ArithmeticError("degenerate design: all lengths are zero")
    s11 = s12 = s22 = r1 = r2 = 0.0
    for l, y in points:
        u = l / l_max
        u2 = u * u
        s11 += u2 * u2
        s12 += u2 * u
        s22 += u2
        r1 += u2 * y
        r2 += u * y
    det = s11 * s22 - s12 * s12
    if not det > 1e-14 * max(s11 * s22, 1e-300):
        raise ArithmeticError("degenerate design: singular normal equations")
    a = (r1 * s22 - r2 * s12) / det / (l_max * l_max)
    b = (s11 * r2 - s12 * r1) / det / l_max
    mean = sum(p[1] for p in points) / len(points)
    ss_res = sum((y - (a * l * l + b * l)) ** 2 for l, y in points)
    ss_tot = sum((y - mean) ** 2 for _, y in points)
    r2v = 1.0 - ss_res / ss_tot if ss_tot > 0 else (1.0 if ss_res == 0 else 0.0)
    return a, b, r2v


def metric_points(records: Sequence[RunRecord], arm: str, metric: str):
    return [(float(r.length), float(r.peak_bytes) if metric == "peak_bytes" else r.seconds)
            for r in records if r.arm == arm]


# ------------------------------------------------------------------ configuration
@dataclass
class ModelConfig:
    d_in: int = 32
    d_z: int = 4
    heads: int = 2
    c: int = 8
    n_query: int = 2
    n_value: int = 2
    rank: int = 2
    precision: str = "f64"
    enforce_head_cap: bool = True

    def validate(self):
        for n in ("d_in", "d_z", "heads", "c", "n_query", "n_value", "rank"):
            if getattr(self, n) < 1:
                raise ValueError(f"{n} must be positive")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision '{self.precision}' (expected f32, f64 or bf16)")
        qk = self.c + 5 * self.n_query + self.rank * self.d_z
        v = self.c + 3 * self.n_value + self.rank * self.d_z
        if self.enforce_head_cap and max(qk, v) > 256:
            raise ValueError(f"lifted head width {max(qk, v)} exceeds the cap of 256")


@dataclass
class DistogramConfig:
    k: int = 20
    n_bins: int = 22
    d_min: float = 2.0
    d_max: float = 22.0
    pe_dim: int = 16


@dataclass
class BenchConfig:
    model: ModelConfig = field(default_factory=ModelConfig)
    distogram: DistogramConfig = field(default_factory=DistogramConfig)
    lengths: List[int] = field(default_factory=list)
    arms: List[str] = field(default_factory=lambda: ["reference", "flash"])
    trials: int = 100
    translation_scale: float = 1.0
    motion_translation_scale: float = 1.0
    tile_rows: int = 64
    tile_cols: int = 64
    reference_byte_budget: int = 1500000000
    threads: int = 1

    def validate(self):
        self.model.validate()
        if not self.arms:
            raise ValueError("at least one arm required")
        for a in self.arms:
            if a not in ARMS:
                raise ValueError(f"unknown arm '{a}' (expected reference or flash)")
        if any(self.lengths[i - 1] >= self.lengths[i] for i in range(1, len(self.lengths))):
            raise ValueError("lengths must be strictly increasing")
        if self.trials < 1:
            raise ValueError("trials must be positive")
        if self.tile_rows < 1 or self.tile_cols < 1:
            raise ValueError("tile sizes must be positive")
        if self.threads < 1:
            raise ValueError("threads must be positive")
        if self.translation_scale < 0 or self.motion_translation_scale < 0:
            raise ValueError("translation scales must be non-negative")


_BENCH_KEYS = ("lengths", "arms", "trials", "translation_scale", "motion_translation_scale", "tile_rows",
               "tile_cols", "reference_byte_budget", "threads")


def load_config(path: str = "") -> BenchConfig:
    """"" = pure defaults; otherwise a JSON file whose omitted fields keep their defaults."""
    cfg = BenchConfig()
    if not path:
        return cfg
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as exc:
        raise IOError(f"cannot open config '{path}'") from exc
    except json.JSONDecodeError as exc:
        raise IOError(f"config '{path}': {exc}") from exc
    try:
        m = j.get("model", {})
        for fld in dataclasses.fields(ModelConfig):
            if fld.name in m:
                setattr(cfg.model, fld.name, type(getattr(cfg.model, fld.name))(m[fld.name]))
        d = j.get("distogram", {})
        for fld in dataclasses.fields(DistogramConfig):
            if fld.name in d:
                setattr(cfg.distogram, fld.name, type(getattr(cfg.distogram, fld.name))(d[fld.name]))
        b = j.get("bench", {})
        for k in _BENCH_KEYS:
            if k in b:
                cur = getattr(cfg, k)
                setattr(cfg, k, list(b[k]) if isinstance(cur, list) else type(cur)(b[k]))
    except (TypeError, ValueError, AttributeError) as exc:
        raise IOError(f"config '{path}': {exc}") from exc
    if cfg.model.precision not in PRECISIONS:
        raise ValueError(f"unknown precision '{cfg.model.precision}'")
    return cfg


def config_to_json(cfg: BenchConfig) -> str:
    j = {"model": dataclasses.asdict(cfg.model), "distogram": dataclasses.asdict(cfg.distogram),
         "bench": {k: getattr(cfg, k) for k in _BENCH_KEYS}}
    return json.dumps(j, separators=(",", ":"), sort_keys=True)  # nlohmann::json dump(): compact, keys sorted


def run_fit(csv_path: str, metric: str, cfg: BenchConfig | None = None) -> RunReport:
    """`fipa fit` (bench.cpp:375-397): refit y = a L^2 + b L per arm of a records CSV."""
    if metric not in ("peak_bytes", "seconds"):
        raise ValueError(f"unknown metric '{metric}' (expected peak_bytes or seconds)")
    rep = RunReport(command="fit", config_echo=config_to_json(cfg or BenchConfig()))
    rep.records = parse_records_csv(csv_path)
    if not rep.records:
        raise ValueError(f"no records found in {csv_path}")
    arms = []
    for r in rep.records:
        if r.arm not in arms:
            arms.append(r.arm)
    for arm in arms:
        a, b, r2 = fit_polynomial(metric_points(rep.records, arm, metric))
        rep.fits.append(FitSummary(arm, metric, a, b, r2))
    return rep


def scaling_checks(report: RunReport, arm: str) -> None:
    """The fits and checks `fipa scaling` attaches per arm (bench.cpp:318-368)."""
    mem = metric_points(report.records, arm, "peak_bytes")
    tim = metric_points(report.records, arm, "seconds")
    if len({p[0] for p in mem}) < 2:
        report.notes.append(f"fits skipped for arm '{arm}': fewer than two measured lengths")
        return
    ma, mb, mr2 = fit_polynomial(mem)
    report.fits.append(FitSummary(arm, "peak_bytes", ma, mb, mr2))
    ta, tb, tr2 = fit_polynomial(tim)
    report.fits.append(FitSummary(arm, "seconds", ta, tb, tr2))
    l_max, peak_at_max = mem[-1]
    if arm == "flash":
        if len(mem) >= 3:
            share = abs(ma) * l_max * l_max / max(peak_at_max, 1.0)
            report.checks.append(CheckOutcome("scaling/flash/quadratic-share", share, 0.01, share < 0.01))
            report.checks.append(CheckOutcome("scaling/flash/memory-fit-r2", mr2, 0.99, mr2 >= 0.99))
        else:
            report.notes.append("flash linearity check skipped: fewer than three measured lengths")
    elif arm == "reference":
        dom = next((p for p in mem if p[0] >= 2048.0), None)
        if dom is not None:
            share = ma * dom[0] * dom[0] / max(dom[1], 1.0)
            report.checks.append(CheckOutcome(f"scaling/reference/quadratic-share@L={int(dom[0])}", share, 0.5,
                                              share > 0.5))
        else:
            report.notes.append("reference quadratic-dominance check skipped: no measured length reaches 2048")


def estimate_reference_bytes(model: ModelConfig, L: int) -> int:
    """bench.cpp:151-155: dense pair tensor plus per-head bias, logits and attention."""
    elt = 8 if model.precision == "f64" else 4
    return (model.d_z + 3 * model.heads) * L * L * elt
