"""BASELINE.md §3 CPU-baseline plan, run on the GPU box's host cores (oracle / bench only).

The UNMODIFIED reference (oracle/_ref/libfipa_ref.so, Release flags) times its own
flash_ipa_forward at f32 storage on the north-star layer shape with threads = 1 and threads =
nproc, using the reference protocol: 1 warm-up, then the median of 3 (proj/src/bench.cpp:285-303).
Each thread count is measured up to the largest L whose single call stays under --budget seconds;
beyond that, y = a L^2 + b L is fitted with the reference's own fit_polynomial
(proj/src/bench.cpp:103-149, called through the compiled library) and the values are reported
as EXTRAPOLATED.  Inputs: reference generators (IpaWeights::init, N(0,1) s/z, random frames).

    python tools/cpu_baseline.py --out profiles/r2_cpu_baseline.json
"""

import argparse
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (north-star shape)
from oracle import fipa_oracle as fo  # noqa: E402
from oracle import ref  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def time_call(cfg, w, p, threads):
    t0 = time.perf_counter()
    ref.flash_forward(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans, None, 64, 64, threads)
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cpu_baseline.json"))
    ap.add_argument("--budget", type=float, default=20.0, help="largest single call measured (s)")
    ap.add_argument("--maxL", type=int, default=65536)
    args = ap.parse_args()
    if not ref.available():
        raise SystemExit("oracle/_ref/libfipa_ref.so missing (build it with make -C oracle)")
    shape = bench.SHAPE
    cfg = fo.IpaConfig(**shape, precision="f32", enforce_head_cap=False)
    w = ref.init_weights(cfg, 0)
    nproc = os.cpu_count() or 1
    result = {"host_cpu": cpu_model(), "host_threads": nproc, "shape": shape, "storage": "f32",
              "protocol": "1 warm-up + median of 3 per point (proj/src/bench.cpp:285-303)", "series": []}
    for threads in (1, nproc):
        pts, rows = [], []
        L = 256
        while L <= args.maxL:
            p = fo.make_problem(cfg, L, 7)
            first = time_call(cfg, w, p, threads)  # warm-up (also the budget probe)
            if first > args.budget:
                break
            ts = [time_call(cfg, w, p, threads) for _ in range(3)]
            med = statistics.median(ts)
            rows.append({"L": L, "seconds": med, "residues_per_s": L / med, "extrapolated": False})
            pts.append((float(L), med))
            print(json.dumps({"threads": threads, **rows[-1]}), flush=True)
            if 4 * med > args.budget:  # the next point (~4x) would exceed the budget
                L *= 2
                break
            L *= 2
        a, b, r2 = ref.fit_polynomial(pts) if len(pts) >= 2 else (0.0, 0.0, 0.0)
        while L <= args.maxL:
            y = a * L * L + b * L
            rows.append({"L": L, "seconds": y, "residues_per_s": L / y if y > 0 else None, "extrapolated": True})
            L *= 2
        result["series"].append({"threads": threads, "fit": {"a": a, "b": b, "r2": r2,
                                                             "model": "seconds = a L^2 + b L (reference fit_polynomial)"},
                                 "points": rows})
    with open(args.out, "w") as f:
        json.dump(result, f, indent=1)
    print(json.dumps({"wrote": args.out}))


if __name__ == "__main__":
    main()
