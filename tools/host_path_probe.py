"""Host-buffer API timing inside a torch process, by chunk size (FIPA_HOST_CHUNK) and phase."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if os.environ.get("PROBE_TORCH", "1") == "1":
    import torch
    t = torch.zeros(10, device="cuda")
import bench
import paper_2505_11580_b200 as fipa
shape = bench.SHAPE
B, L = 8, 1024
m = fipa.Model(**shape, precision="bf16", seed=0, enforce_head_cap=False)
h = bench.synth_inputs(B, L, shape)
a64 = [h[k].astype(np.float64) for k in ("s", "z1", "z2", "rot", "trans")]
d64 = np.random.default_rng(0).standard_normal((B, L, shape["d_in"]))
for name, fn in (("fwd", lambda: m.flash(*a64, mask=h["mask"])), ("grad", lambda: m.flash_grad(*a64, d64, mask=h["mask"]))):
    fn()
    ts = []
    for _ in range(7):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    print(os.environ.get("FIPA_HOST_CHUNK", "auto"), "torch" if "torch" in sys.modules else "no-torch", name,
          "median ms %.2f" % (np.median(ts) * 1e3))
t0 = time.perf_counter(); z = np.empty((B, L, 1036)); z.fill(1.0); print("alloc+touch 68MB ms %.2f" % ((time.perf_counter() - t0) * 1e3))
