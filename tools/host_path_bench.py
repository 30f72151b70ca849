"""Time the host-buffer API (Model.flash / flash_grad) at B=8 L=1024: float64 and float32 arrays."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench
import paper_2505_11580_b200 as fipa

shape = bench.SHAPE
B, L = int(os.environ.get("HB", 8)), int(os.environ.get("HL", 1024))
m = fipa.Model(**shape, precision="bf16", seed=0, enforce_head_cap=False)
h = bench.synth_inputs(B, L, shape)
a64 = [h[k].astype(np.float64) for k in ("s", "z1", "z2", "rot", "trans")]
a32 = [h[k] for k in ("s", "z1", "z2", "rot", "trans")]
d64 = np.random.default_rng(0).standard_normal((B, L, shape["d_in"]))
d32 = d64.astype(np.float32)
print("cpus", os.cpu_count())
t = time.perf_counter(); x = a64[0].astype(np.float32); print("numpy s f64->f32 %.2f ms" % ((time.perf_counter() - t) * 1e3))
for name, fn in (("flash f64", lambda: m.flash(*a64, mask=h["mask"])), ("flash f32", lambda: m.flash(*a32, mask=h["mask"])),
                 ("grad f64", lambda: m.flash_grad(*a64, d64, mask=h["mask"])),
                 ("grad f32", lambda: m.flash_grad(*a32, d32, mask=h["mask"]))):
    fn(); fn()
    ts = []
    for _ in range(5):
        t = time.perf_counter(); fn(); ts.append(time.perf_counter() - t)
    med = float(np.median(ts))
    print(f"{name}: {med*1e3:.2f} ms  {B*L/med/1e6:.2f} M residues/s", flush=True)
