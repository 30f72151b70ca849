"""`fipa scaling` / `fipa fit` on the GPU (reference proj/src/bench.cpp:251-397).

scaling: for each arm ("reference" = the quadratic-memory dense forward, Model.reference_device;
"flash" = the linear-memory layer, Model.forward_device) and each L, one layer forward over B=1
synthetic inputs: peak_bytes = the device bytes the call needs (its workspace + output -- what the
reference's allocation ledger counts inside the forward), seconds = median of 3 device-timed runs
(CUDA events) after one warm-up (bench.cpp:285-303).  The quadratic arm is skipped where its
workspace exceeds `reference_byte_budget` (bench.cpp:263-272).  Fits y = a L^2 + b L and the
reference's linearity / dominance checks are attached; the report is the reference's CSV / JSON
schema (paper_2505_11580_b200/report.py), so it can be refit with `fit` and diffed against CPU
records of the reference.

    python tools/scaling.py scaling --config cfg.json --lengths 256,512,...,16384 --format json --out r.json
    python tools/scaling.py fit records.csv --metric seconds
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_11580_b200 import report as rp  # noqa: E402

MAIN = dict(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2)


def run_scaling(cfg: rp.BenchConfig, seed: int, flash_precision: str) -> rp.RunReport:
    import numpy as np
    import torch

    import bench
    import paper_2505_11580_b200 as fipa

    cfg.validate()
    rep = rp.RunReport(command="scaling", config_echo=rp.config_to_json(cfg))
    lengths = cfg.lengths or [128, 256, 512, 1024, 2048, 4096, 8192]
    shape = {k: getattr(cfg.model, k) for k in ("d_in", "d_z", "heads", "c", "n_query", "n_value", "rank")}
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    for arm in cfg.arms:
        precision = flash_precision if arm == "flash" else "f32"
        model = fipa.Model(**shape, precision=precision, seed=seed, enforce_head_cap=cfg.model.enforce_head_cap)
        for L in lengths:
            out_bytes = L * shape["d_in"] * 4
            ws_bytes = model.reference_workspace_size(1, L) if arm == "reference" else model.workspace_size(1, L)
            if arm == "reference" and ws_bytes + out_bytes > cfg.reference_byte_budget:
                note = (f"reference arm skipped at L={L}: estimated peak {ws_bytes + out_bytes} bytes exceeds "
                        f"budget {cfg.reference_byte_budget}")
                rep.notes.append(note)
                print("warning: " + note, file=sys.stderr)
                continue
            host = bench.synth_inputs(1, L, shape, seed=seed + L)
            t = {k: torch.from_numpy(v).to(dev) for k, v in host.items()}
            out = torch.empty((1, L, shape["d_in"]), dtype=torch.float32, device=dev)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            p = {k: v.data_ptr() for k, v in t.items()}
            fn = model.reference_device if arm == "reference" else model.forward_device

            def call():
                fn(1, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(), ws.data_ptr(),
                   ws_bytes, st.cuda_stream)

            call()  # warm-up
            secs = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                call()
                b.record(st)
                b.synchronize()
                secs.append(a.elapsed_time(b) / 1e3)
            assert bool(torch.isfinite(out).all().item())
            rep.records.append(rp.RunRecord(arm, L, seed, precision, int(ws_bytes + out_bytes),
                                            float(np.median(secs))))
            print(f"{arm:9s} L={L:6d} {precision} peak={ws_bytes + out_bytes:>14d} B  {np.median(secs) * 1e3:9.3f} ms",
                  file=sys.stderr, flush=True)
            del ws, out, t
            torch.cuda.empty_cache()
        rp.scaling_checks(rep, arm)
    return rep


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    sc = sub.add_parser("scaling")
    sc.add_argument("--config", default="")
    sc.add_argument("--main-shape", action="store_true", help="north-star layer shape instead of the config's model")
    sc.add_argument("--lengths", default="")
    sc.add_argument("--seed", type=int, default=0)
    sc.add_argument("--budget", type=float, default=0, help="reference_byte_budget override (bytes)")
    sc.add_argument("--flash-precision", default="bf16", choices=["bf16", "f32"])
    sc.add_argument("--format", default="json", choices=["json", "csv"])
    sc.add_argument("--out", default="-")
    ft = sub.add_parser("fit")
    ft.add_argument("csv")
    ft.add_argument("--metric", default="seconds", choices=["seconds", "peak_bytes"])
    ft.add_argument("--config", default="")
    ft.add_argument("--format", default="json", choices=["json", "csv"])
    ft.add_argument("--out", default="-")
    args = ap.parse_args()
    cfg = rp.load_config(args.config)
    if args.cmd == "fit":
        rep = rp.run_fit(args.csv, args.metric, cfg)
    else:
        if args.main_shape:
            for k, v in MAIN.items():
                setattr(cfg.model, k, v)
            cfg.model.enforce_head_cap = False
            cfg.model.precision = "f32"
        if args.lengths:
            cfg.lengths = [int(x) for x in args.lengths.split(",")]
        if args.budget:
            cfg.reference_byte_budget = int(args.budget)
        rep = run_scaling(cfg, args.seed, args.flash_precision)
    rp.emit_report(rep, args.format, args.out)
    return 0 if rep.all_pass() else 1


if __name__ == "__main__":
    sys.exit(main())
