"""Materialised (z_factor_rank 3-4) backward: per-gradient deviation from the oracle at a small
shape, and the training-step time at B=8 L=1024 (device, graph replay) -- run on a GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import paper_2505_11580_b200 as fipa  # noqa: E402
from helpers import MAIN, gpu_train_device, make_batch, oracle_backward, oracle_weights_for, rel_dev  # noqa: E402
from oracle import fipa_oracle as fo  # noqa: E402

GRADS = ("s", "z1", "z2", "rot", "trans") + fo.WEIGHT_NAMES
for rank in (3, 4):
    shape = dict(MAIN, rank=rank)
    m = fipa.Model(**shape, precision="bf16", seed=3, enforce_head_cap=False)
    batch = make_batch(shape, 2, 200, seed=3, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(3).standard_normal((2, 200, shape["d_in"]))
    g = gpu_train_device(m, batch, dout)[1]
    ref = oracle_backward(shape, oracle_weights_for(m, "bf16"), batch, dout)
    print("rank", rank, "max dev", " ".join(f"{n}={rel_dev(ref[n], g[n]):.1e}" for n in GRADS), flush=True)

import bench  # noqa: E402
dev = torch.device("cuda:0")
for rank in (2, 3, 4):
    shape = dict(bench.SHAPE, rank=rank)
    B, L = 8, 1024
    m = fipa.Model(**shape, precision="bf16", seed=0, enforce_head_cap=False)
    h = bench.synth_inputs(B, L, shape)
    t = {k: torch.from_numpy(v).to(dev) for k, v in h.items()}
    out = torch.empty((B, L, shape["d_in"]), device=dev)
    dout = torch.randn((B, L, shape["d_in"]), device=dev)
    g = {k: torch.empty_like(t[k]) for k in ("s", "z1", "z2", "rot", "trans")}
    gw = torch.empty(m.num_weights(), device=dev)
    nb = m.train_workspace_size(B, L)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    p = {k: v.data_ptr() for k, v in t.items()}

    def step():
        m.forward_train_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(),
                               ws.data_ptr(), nb, st)
        m.backward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], dout.data_ptr(),
                          g["s"].data_ptr(), g["z1"].data_ptr(), g["z2"].data_ptr(), g["rot"].data_ptr(),
                          g["trans"].data_ptr(), gw.data_ptr(), ws.data_ptr(), nb, st)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"rank {rank} B={B} L={L} fwd+bwd {ms:.3f} ms/step = {B * L / ms * 1e3 / 1e6:.2f} M residues/s, "
          f"workspace {nb / 2**20:.0f} MiB", flush=True)
