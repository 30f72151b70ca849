"""Per-kernel summary (JSON) of an `ncu --set full` report: duration, DRAM bytes, tensor-pipe and
SM throughput, grid -- the numbers the profiles/ summaries and bench.py's roofline `traffic` cite.

    python tools/ncu_summary.py report.ncu-rep "command that produced it" "workload" > out.json
"""
import csv
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": ("duration_us_under_ncu", 1e-3),
    "dram__bytes_read.sum": ("dram_read_MB", 1e-6),
    "dram__bytes_write.sum": ("dram_write_MB", 1e-6),
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": ("tensor_active_pct", 1.0),
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": ("sm_throughput_pct", 1.0),
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("dram_throughput_pct", 1.0),
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": ("dram_throughput_pct", 1.0),
    "launch__grid_size": ("grid", 1.0),
    "smsp__cycles_active.avg.per_second": ("sm_clock_ghz", 1e-9),
}
UNIT_SCALE = {"ns": 1.0, "us": 1e3, "ms": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
              "KB": 1e3, "MB": 1e6, "GB": 1e9, "cycle/second": 1.0, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
              "%": 1.0, "": 1.0}


def main():
    rep, cmd, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    # section-prefixed names ("TPC.TriageCompute.<metric>") -> bare metric names
    head = [h.split(".", 2)[-1] if h.count(".") >= 2 and h.split(".")[0].isupper() else h for h in rows[0]]
    units = rows[1]
    ki = head.index("Kernel Name")
    kernels = []
    for r in rows[2:]:
        if len(r) != len(head):
            continue
        k = {"kernel": r[ki][:120]}
        for m, (name, scale) in WANT.items():
            if m not in head:
                continue
            i = head.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            k[name] = v * UNIT_SCALE.get(units[i], 1.0) * scale if m != "launch__grid_size" else int(v)
        kernels.append(k)
    print(json.dumps({"command": cmd, "workload": workload,
                      "note": "cold-cache, serialised replays: per-kernel shares, not bench timings",
                      "kernels": kernels}, indent=1))


if __name__ == "__main__":
    main()
