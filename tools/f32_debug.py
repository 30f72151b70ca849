import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import paper_2505_11580_b200 as fipa
from helpers import MAIN, TINY, make_batch, oracle_forward, oracle_weights_for, rel_dev, gpu_forward_device, ws_view, oracle_cfg
from oracle import fipa_oracle as fo

for shape in (TINY, MAIN):
    B, L = 1, 130
    model = fipa.Model(**shape, precision="f32", seed=3, enforce_head_cap=False)
    w = oracle_weights_for(model, "f32")
    batch = make_batch(shape, B, L, seed=5)
    res = {}
    for tc in (True, False):
        model.set_tuning(f32_tc=tc)
        out, ws, ((off, dims)) = gpu_forward_device(model, batch)
        n_proj, dqk_pad, dv_pad, nfeat = dims
        H = shape["heads"]
        proj = ws_view(ws, off[2], B * L * n_proj, "f32").reshape(B * L, n_proj)
        q = ws_view(ws, off[3], H * L * dqk_pad, "f32").reshape(H, L, dqk_pad)
        feat = ws_view(ws, off[8], B * L * nfeat, "f32").reshape(B * L, nfeat)
        lse = ws_view(ws, off[7], H * L, "f32")
        res[tc] = dict(out=out, proj=proj, q=q, feat=feat, lse=lse)
    for k in res[True]:
        print(shape["d_in"], k, rel_dev(res[False][k], res[True][k]))
    a, b = res[False]["feat"], res[True]["feat"]
    seg = shape["d_z"] + shape["c"] + 4 * shape["n_value"]
    err = np.abs(a - b).reshape(B * L, H, seg).max(axis=(0, 1))
    print("feat err by column within seg:", np.round(err / np.abs(a).max(), 4))
    errr = np.abs(a - b).max(axis=1)
    print("feat err by row (first 20):", np.round(errr[:20] / np.abs(a).max(), 4), "rows>1e-3:", np.nonzero(errr / np.abs(a).max() > 1e-3)[0][:20])
    ea = np.abs(res[False]["out"] - res[True]["out"]).reshape(B * L, -1).max(axis=1)
    print("out err rows:", np.nonzero(ea > 1e-3 * np.abs(res[False]["out"]).max())[0][:20])
