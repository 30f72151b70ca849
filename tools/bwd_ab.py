"""A/B of attention-backward ring plans at B=8 L=1024 (stage times of the training step).
usage: python tools/bwd_ab.py "1,6,2,0,16" "1,3,2,0,32" ..."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench
import paper_2505_11580_b200 as fipa

shape = bench.SHAPE
B, L = int(os.environ.get("AB_B", 8)), int(os.environ.get("AB_L", 1024))
dev = torch.device("cuda:0")
m = fipa.Model(**shape, precision="bf16", seed=0, enforce_head_cap=False)
h = bench.synth_inputs(B, L, shape)
t = {k: torch.from_numpy(v).to(dev) for k, v in h.items()}
out = torch.empty((B, L, shape["d_in"]), device=dev)
dout = torch.randn((B, L, shape["d_in"]), device=dev)
g = {k: torch.empty_like(t[k]) for k in ("s", "z1", "z2", "rot", "trans")}
gw = torch.empty(m.num_weights(), device=dev)
nb = m.train_workspace_size(B, L)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
p = {k: v.data_ptr() for k, v in t.items()}
names = ["dout", "dfeat", "dw_out", "prep", "dkdv", "dq", "unpack", "recenter", "ds", "dW", "scatter"]
ref = None
for cfg in sys.argv[1:]:
    ring = [int(x) for x in cfg.split(",")]
    ds = int(os.environ.get("AB_DS", -1))
    m.set_tuning(bwd_ring=ring, bwd_ds=ds)
    def step():
        m.forward_train_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(),
                               ws.data_ptr(), nb, st)
        m.backward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], dout.data_ptr(),
                          g["s"].data_ptr(), g["z1"].data_ptr(), g["z2"].data_ptr(), g["rot"].data_ptr(),
                          g["trans"].data_ptr(), gw.data_ptr(), ws.data_ptr(), nb, st)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    m.set_timing(True)
    rows = []
    for _ in range(10):
        flush.zero_()
        step()
        torch.cuda.synchronize()
        rows.append(m.bwd_stage_times())
    m.set_timing(False)
    med = np.median(np.array(rows), 0)
    cur = torch.cat([g["s"].flatten(), g["rot"].flatten(), gw]).cpu().numpy()
    if ref is None:
        ref = cur
    err = np.abs(cur - ref).max() / np.abs(ref).max()
    print(cfg, "ds", ds, " ".join(f"{n}={v:.4f}" for n, v in zip(names, med)), f"total_bwd={med.sum():.4f} dev_vs_first={err:.2e}",
          flush=True)
