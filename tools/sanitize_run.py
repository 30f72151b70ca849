"""Small-L workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
of the layer once -- forward (CTA pair, two-pass, single CTA, 3xTF32), training forward + backward
(materialised dS and streaming dQ), the sharded blocks, the producer, the dense arm."""
import os, sys
import numpy as np
import torch
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2505_11580_b200 as fipa
from helpers import MAIN, make_batch, gpu_forward_device, gpu_train_device

which = sys.argv[1] if len(sys.argv) > 1 else "all"
B, L = 1, 256
batch = make_batch(MAIN, B, L, seed=1, mask_frac=0.1, bf16=True)
dout = np.random.default_rng(0).standard_normal((B, L, MAIN["d_in"]))
if which in ("all", "fwd"):
    m = fipa.Model(**MAIN, precision="bf16", seed=0, enforce_head_cap=False)
    for impl in ("pair", "pass", "1sm"):
        m.set_tuning(attn_impl=impl)
        gpu_forward_device(m, batch)
    m.set_tuning(attn_impl="auto", fused_pack=False)
    gpu_forward_device(m, batch)
    print("fwd ok", flush=True)
if which in ("all", "bwd"):
    m = fipa.Model(**MAIN, precision="bf16", seed=0, enforce_head_cap=False)
    for ds in (1, 0):
        m.set_tuning(bwd_ds=ds)
        gpu_train_device(m, batch, dout)
    # query-chunked dS (two 256-query chunks: TMA-reduction accumulators) and the micro-batched capture
    b2 = make_batch(MAIN, 2, 512, seed=2, mask_frac=0.1, bf16=True)
    d2 = np.random.default_rng(1).standard_normal((2, 512, MAIN["d_in"]))
    m.set_tuning(bwd_ds=-1, ds_cap_mb=4, micro=2)
    gpu_train_device(m, b2, d2)
    # whole-query materialised dS with the micro-batched capture (bf16 dQ / dK / dV hand-off)
    m.set_tuning(ds_cap_mb=2048)
    gpu_train_device(m, b2, d2)
    print("bwd ok", flush=True)
if which in ("all", "wide"):
    # z_factor_rank 3: the materialised backward (batched GEMMs + streaming softmax kernels)
    r3 = dict(MAIN, rank=3)
    m = fipa.Model(**r3, precision="bf16", seed=0, enforce_head_cap=False)
    b3 = make_batch(r3, 2, 192, seed=5, mask_frac=0.1, bf16=True)
    gpu_train_device(m, b3, np.random.default_rng(5).standard_normal((2, 192, r3["d_in"])))
    print("wide ok", flush=True)
if which in ("all", "f32"):
    m = fipa.Model(**MAIN, precision="f32", seed=0, enforce_head_cap=False)
    gpu_forward_device(m, batch)
    print("f32 ok", flush=True)
if which in ("all", "misc"):
    r3 = dict(MAIN, rank=3)
    m = fipa.Model(**r3, precision="bf16", seed=0, enforce_head_cap=False)
    gpu_forward_device(m, make_batch(r3, 1, 200, seed=2, bf16=True))
    fipa.knn_distogram(np.random.default_rng(0).standard_normal((1, 100, 3)), k=8)
    m = fipa.Model(seed=0)
    m.reference(*[make_batch(dict(d_in=32, d_z=4, heads=2, c=8, n_query=2, n_value=2, rank=2), 1, 40, seed=3)[k][0]
                  for k in ("s", "z1", "z2", "rot", "trans")])
    print("misc ok", flush=True)
torch.cuda.synchronize()
