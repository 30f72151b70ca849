"""GPU check of the fp32-accuracy path (3xTF32 tensor cores vs the CUDA-core kernels vs the oracle)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import paper_2505_11580_b200 as fipa  # noqa: E402
from helpers import MAIN, TINY, make_batch, oracle_forward, oracle_weights_for, rel_dev, gpu_forward_device  # noqa: E402

for shape, B, L, scale in ((TINY, 2, 77, 1.0), (MAIN, 2, 300, 1.0), (MAIN, 1, 700, 30.0), (MAIN, 8, 1024, 1.0)):
    model = fipa.Model(**shape, precision="f32", seed=3, enforce_head_cap=False)
    w = oracle_weights_for(model, "f32")
    batch = make_batch(shape, B, L, seed=5, translation_scale=scale, mask_frac=0.1)
    res = {}
    for tc in (True, False):
        model.set_tuning(f32_tc=tc)
        out, _, _ = gpu_forward_device(model, batch)
        import torch
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            gpu_forward_device(model, batch)
        res[tc] = (out, (time.perf_counter() - t0) / 3, model.forward_launches())
    ref = oracle_forward(shape, w, batch) if L <= 700 else None
    print(f"shape d_in={shape['d_in']} B={B} L={L} scale={scale}: tc vs simt {rel_dev(res[False][0], res[True][0]):.3e}",
          f"tc vs oracle {rel_dev(ref, res[True][0]) if ref is not None else float('nan'):.3e}",
          f"simt vs oracle {rel_dev(ref, res[False][0]) if ref is not None else float('nan'):.3e}",
          f"launches {res[True][2]}/{res[False][2]} wall(incl copies) {res[True][1]*1e3:.2f}/{res[False][1]*1e3:.2f} ms",
          flush=True)
