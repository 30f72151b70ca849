"""BASELINE cfg5: FlashIPA layer forward sweep over L (and z_factor_rank) on one B200.

For each (rank, L): device time of one layer forward (CUDA events, median of 5 after 2 warm-ups,
L2 flushed before each), residues/s, attention-equivalent TFLOP/s (2*B*H*L^2*(D_qk+D_v) over the
whole layer time), and the device memory the call needs (workspace bytes + inputs/outputs) to
show memory linear in L.  Every rank runs the bf16 tcgen05 path: rank 1-2 the CTA-pair kernel,
rank 3-4 (lifted widths 560-704) the two-pass CTA-pair kernel (attn_fwd_pass.cu).

    python tools/sweep.py --out profiles/r2_sweep.json   (each row carries the SM clocks sampled
    during its timed reps)
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (synthetic inputs, flop counts)
import paper_2505_11580_b200 as fipa  # noqa: E402


def run(shape, precision, B, L, reps=5):
    dev = torch.device("cuda:0")
    model = fipa.Model(**shape, precision=precision, seed=0, enforce_head_cap=False)
    host = bench.synth_inputs(B, L, shape, seed=7)
    t = {k: torch.from_numpy(v).to(dev) for k, v in host.items()}
    out = torch.empty((B, L, shape["d_in"]), dtype=torch.float32, device=dev)
    nbytes = model.workspace_size(B, L)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    p = {k: v.data_ptr() for k, v in t.items()}

    def step():
        model.forward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(),
                             ws.data_ptr(), nbytes, st.cuda_stream)

    for _ in range(2):
        step()
    # enough reps that the clock sampler sees the timed region (>= ~30 ms in total)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    step()
    b.record(st)
    b.synchronize()
    reps = max(reps, min(400, int(30.0 / max(a.elapsed_time(b), 1e-3))))
    times = []
    with bench.ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            step()
            b.record(st)
            b.synchronize()
            times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    ok = bool(torch.isfinite(out).all().item())
    io = sum(v.numel() * v.element_size() for v in t.values()) + out.numel() * 4
    return {"rank": shape["rank"], "precision": precision, "B": B, "L": L, "ms": ms,
            "residues_per_s": B * L / (ms / 1e3),
            "attn_equiv_tflops": bench.attn_flops(shape, B, L) / (ms / 1e3) / 1e12,
            "workspace_bytes": nbytes, "device_bytes_total": nbytes + io,
            "bytes_per_residue": (nbytes + io) / (B * L), "finite": ok, "clocks": clk.summary(),
            "l2": "flushed (256 MiB write) before every rep"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_sweep.json"))
    ap.add_argument("--maxL", type=int, default=65536)
    ap.add_argument("--minL", type=int, default=256)
    ap.add_argument("--ranks", default="1,2,3,4")
    args = ap.parse_args()
    rows = []
    for r in [int(x) for x in args.ranks.split(",")]:
        shape = dict(bench.SHAPE, rank=r)
        L = args.minL
        while L <= args.maxL:
            rows.append(run(shape, "bf16", 1, L))
            print(json.dumps(rows[-1]), flush=True)
            L *= 2
    with open(args.out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
