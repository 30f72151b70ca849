"""GPU: query-row sharding (BASELINE cfg4 path).  Only one GPU is available to the tests, so the
G-rank decomposition is driven through the collective-agnostic C-ABI building blocks
(shard_centroid_sums / shard_pack / shard_attend) with the all-reduce and the rank-major
all-gather done by device copies on one GPU; the NCCL path itself runs at world size 1."""

import numpy as np
import pytest
import torch

from helpers import BF16_TOL, MAIN, gpu_forward_device, make_batch, oracle_forward, oracle_weights_for, rel_dev
from paper_2505_11580_b200 import sharding

pytestmark = pytest.mark.gpu


def _dev(batch):
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(batch[k], dtype=np.float32)).to(dev)
         for k in ("s", "z1", "z2", "rot", "trans")}
    t["mask"] = torch.from_numpy(np.ascontiguousarray(batch["mask"], dtype=np.uint8)).to(dev)
    return t


@pytest.mark.parametrize("G,B,rank", [(2, 1, 2), (4, 2, 2), (2, 1, 3)])
def test_emulated_shards_match_unsharded_forward(fipa, G, B, rank):
    shape = dict(MAIN, rank=rank)  # rank 3: the two-pass attention kernel reads the sharded keys
    model = fipa.Model(**shape, precision="bf16", seed=3, enforce_head_cap=False)
    L = 128 * G
    batch = make_batch(shape, B, L, seed=31, mask_frac=0.1, bf16=True)
    ref_gpu, _, _ = gpu_forward_device(model, batch)
    t = _dev(batch)
    st = torch.cuda.current_stream().cuda_stream
    n = L // G
    shards, sums = [], torch.zeros(B * 4, dtype=torch.float32, device="cuda")
    for r in range(G):
        lo, hi = sharding.row_block(L, G, r)
        sh = {k: v[:, lo:hi].contiguous() for k, v in t.items()}
        sh["ws"] = torch.zeros(model.workspace_size(B, n), dtype=torch.uint8, device="cuda")
        part = torch.zeros(B * 4, dtype=torch.float32, device="cuda")
        model.shard_centroid_sums(B, n, sh["trans"].data_ptr(), sh["mask"].data_ptr(), part.data_ptr(), st)
        sums += part  # the all-reduce
        shards.append(sh)
    k_all = v_all = None
    for r, sh in enumerate(shards):
        kp, kb, vp, vb = model.shard_pack(B, n, sh["s"].data_ptr(), sh["z1"].data_ptr(), sh["z2"].data_ptr(),
                                          sh["rot"].data_ptr(), sh["trans"].data_ptr(), sh["mask"].data_ptr(),
                                          sums.data_ptr(), sh["ws"].data_ptr(), sh["ws"].numel(), st)
        if k_all is None:
            k_all = torch.empty((G, kb), dtype=torch.uint8, device="cuda")
            v_all = torch.empty((G, vb), dtype=torch.uint8, device="cuda")
        base = sh["ws"].data_ptr()
        k_all[r].copy_(sh["ws"][kp - base:kp - base + kb])  # the rank-major all-gather
        v_all[r].copy_(sh["ws"][vp - base:vp - base + vb])
    outs = []
    for r, sh in enumerate(shards):
        out = torch.empty((B, n, MAIN["d_in"]), dtype=torch.float32, device="cuda")
        model.shard_attend(B, n, G, sh["s"].data_ptr(), sh["z1"].data_ptr(), sh["z2"].data_ptr(),
                           sh["rot"].data_ptr(), sh["trans"].data_ptr(), sh["mask"].data_ptr(), k_all.data_ptr(),
                           v_all.data_ptr(), out.data_ptr(), sh["ws"].data_ptr(), sh["ws"].numel(), st)
        outs.append(out)
    torch.cuda.synchronize()
    got = torch.cat(outs, 1).cpu().numpy().astype(np.float64)
    assert rel_dev(ref_gpu, got) < 1e-3  # only the centroid's summation order differs
    ref = oracle_forward(shape, oracle_weights_for(model, "bf16"), batch)
    assert rel_dev(ref, got) < BF16_TOL


def test_nccl_world1_gradient_all_reduce_is_identity(fipa):
    comm = fipa.Comm(1, 0, fipa.comm_unique_id(), 0)
    buf = torch.randn(1 << 20, dtype=torch.float32, device="cuda")
    ref = buf.clone()
    comm.all_reduce_sum_f32(buf.data_ptr(), buf.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)


def test_nccl_world1_sharded_forward_equals_forward(fipa):
    model = fipa.Model(**MAIN, precision="bf16", seed=4, enforce_head_cap=False)
    B, L = 1, 192
    batch = make_batch(MAIN, B, L, seed=41, mask_frac=0.1, bf16=True)
    ref_gpu, _, _ = gpu_forward_device(model, batch)
    t = _dev(batch)
    comm = fipa.Comm(1, 0, fipa.comm_unique_id(), 0)
    ws = torch.zeros(model.sharded_workspace_size(B, L, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, L, MAIN["d_in"]), dtype=torch.float32, device="cuda")
    model.forward_sharded_device(comm, B, L, t["s"].data_ptr(), t["z1"].data_ptr(), t["z2"].data_ptr(),
                                 t["rot"].data_ptr(), t["trans"].data_ptr(), t["mask"].data_ptr(), out.data_ptr(),
                                 ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    # identical kernels; only the centroid (all-reduced partial sums vs one block) rounds differently
    assert rel_dev(ref_gpu, out.cpu().numpy().astype(np.float64)) < 1e-3
