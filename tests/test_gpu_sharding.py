"""GPU: query-row sharding (BASELINE cfg4 path).  Only one GPU is available to the tests, so the
G-rank decomposition is driven through the collective-agnostic C-ABI building blocks
(shard_centroid_sums / shard_pack / shard_attend) with the all-reduce and the rank-major
all-gather done by device copies on one GPU; the NCCL path itself runs at world size 1."""

import numpy as np
import pytest
import torch

from helpers import BF16_TOL, MAIN, gpu_forward_device, make_batch, oracle_forward, oracle_weights_for, rel_dev
from oracle import fipa_oracle as fo
from paper_2505_11580_b200 import sharding

pytestmark = pytest.mark.gpu


def _dev(batch):
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(batch[k], dtype=np.float32)).to(dev)
         for k in ("s", "z1", "z2", "rot", "trans")}
    t["mask"] = torch.from_numpy(np.ascontiguousarray(batch["mask"], dtype=np.uint8)).to(dev)
    return t


@pytest.mark.parametrize("G,B,rank,n_local", [(2, 1, 2, 128), (4, 2, 2, 128), (2, 1, 3, 128), (8, 1, 2, 2048)])
def test_emulated_shards_match_unsharded_forward(fipa, G, B, rank, n_local):
    """G query-row shards through the C-ABI blocks (centroid sums -> pack -> rank-major gather ->
    attend) against the unsharded forward; up to L = 16384 over 8 shards (the cfg4 regime; the
    oracle comparison only at the small sizes)."""
    shape = dict(MAIN, rank=rank)  # rank 3: the two-pass attention kernel reads the sharded keys
    model = fipa.Model(**shape, precision="bf16", seed=3, enforce_head_cap=False)
    L = n_local * G
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
    if L <= 1024:
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


@pytest.mark.parametrize("chunks", [2, 4])
def test_nccl_world1_overlapped_gather_equals_single_gather(fipa, chunks):
    """The head-chunked gather / attention overlap (K/V rows sent in head chunks on a side stream,
    attention of chunk c launched once its keys landed, output GEMM after the last) gives the same
    output, bit for bit, as one all-gather followed by one attention launch."""
    model = fipa.Model(**MAIN, precision="bf16", seed=6, enforce_head_cap=False)
    B, L = 2, 256
    batch = make_batch(MAIN, B, L, seed=61, mask_frac=0.1, bf16=True)
    t = _dev(batch)
    comm = fipa.Comm(1, 0, fipa.comm_unique_id(), 0)
    outs = {}
    for c in (1, chunks):
        model.set_tuning(shard_chunks=c)
        assert model.tuning()["shard_chunks"] == c
        ws = torch.zeros(model.sharded_workspace_size(B, L, 1), dtype=torch.uint8, device="cuda")
        out = torch.empty((B, L, MAIN["d_in"]), dtype=torch.float32, device="cuda")
        model.forward_sharded_device(comm, B, L, t["s"].data_ptr(), t["z1"].data_ptr(), t["z2"].data_ptr(),
                                     t["rot"].data_ptr(), t["trans"].data_ptr(), t["mask"].data_ptr(),
                                     out.data_ptr(), ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs[c] = out.cpu().numpy()
    assert np.array_equal(outs[1], outs[chunks])


@pytest.mark.parametrize("n", [256, 1024])
def test_emulated_sharded_training_matches_unsharded(fipa, n):
    """Query-row-sharded training step for G=2 ranks emulated on one GPU through the
    collective-agnostic C-ABI blocks: all-reduce of centroid sums, all-gather of packed keys,
    reduce-scatter of the partial key gradients, all-reduce of the translation-gradient sums and of
    the weight gradients.  Output and every gradient must match the unsharded training step (which
    at L = 2048 takes the materialised-dS path, while the shards run the streaming dQ kernel), and
    at L_local = 1024 the oracle-equivalent checker as well."""
    from helpers import emulated_backward, gpu_train_device

    G, B = 2, 1
    L = G * n
    model = fipa.Model(**MAIN, precision="bf16", seed=12, enforce_head_cap=False)
    batch = make_batch(MAIN, B, L, seed=57, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(5).standard_normal((B, L, MAIN["d_in"]))
    ref_out, ref_g, _, _ = gpu_train_device(model, batch, dout)

    t = _dev(batch)
    t["dout"] = torch.from_numpy(dout.astype(np.float32)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    H, rdz, din = MAIN["heads"], MAIN["rank"] * MAIN["d_z"], MAIN["d_in"]
    nw = model.num_weights()
    ranks, sums = [], torch.zeros(B * 4, dtype=torch.float32, device="cuda")
    for r in range(G):
        lo, hi = sharding.row_block(L, G, r)
        sh = {k: v[:, lo:hi].contiguous() for k, v in t.items()}
        sh["ws"] = torch.zeros(model.train_workspace_size(B, n), dtype=torch.uint8, device="cuda")
        part = torch.zeros(B * 4, dtype=torch.float32, device="cuda")
        model.shard_centroid_sums(B, n, sh["trans"].data_ptr(), sh["mask"].data_ptr(), part.data_ptr(), st)
        sums += part  # all-reduce
        ranks.append(sh)
    p = lambda sh, k: sh[k].data_ptr()  # noqa: E731
    k_all = v_all = None
    for r, sh in enumerate(ranks):
        kp, kb, vp, vb = model.shard_pack(B, n, p(sh, "s"), p(sh, "z1"), p(sh, "z2"), p(sh, "rot"), p(sh, "trans"),
                                          p(sh, "mask"), sums.data_ptr(), p(sh, "ws"), sh["ws"].numel(), st,
                                          train=True)
        if k_all is None:
            k_all = torch.empty((G, kb), dtype=torch.uint8, device="cuda")
            v_all = torch.empty((G, vb), dtype=torch.uint8, device="cuda")
        base = sh["ws"].data_ptr()
        k_all[r].copy_(sh["ws"][kp - base:kp - base + kb])  # all-gather (rank-major)
        v_all[r].copy_(sh["ws"][vp - base:vp - base + vb])
    outs = []
    for sh in ranks:
        sh["out"] = torch.empty((B, n, din), dtype=torch.float32, device="cuda")
        model.shard_attend(B, n, G, p(sh, "s"), p(sh, "z1"), p(sh, "z2"), p(sh, "rot"), p(sh, "trans"),
                           p(sh, "mask"), k_all.data_ptr(), v_all.data_ptr(), p(sh, "out"), p(sh, "ws"),
                           sh["ws"].numel(), st, train=True)
        outs.append(sh["out"])
    part_n = B * n * H * 448
    for sh in ranks:
        sh["dk_part"] = torch.zeros(G * part_n, dtype=torch.float32, device="cuda")
        sh["dv_part"] = torch.zeros(G * part_n, dtype=torch.float32, device="cuda")
        sh["dk_own"] = torch.zeros(part_n, dtype=torch.float32, device="cuda")
        sh["dv_own"] = torch.zeros(part_n, dtype=torch.float32, device="cuda")
        sh["dt_sums"] = torch.zeros(B * 4, dtype=torch.float32, device="cuda")
        for k, shape in (("ds", (B, n, din)), ("dz1", (B, n, MAIN["rank"], MAIN["d_z"])),
                         ("dz2", (B, n, MAIN["rank"], MAIN["d_z"])), ("drot", (B, n, 3, 3)), ("dtrans", (B, n, 3))):
            sh[k] = torch.full(shape, float("nan"), dtype=torch.float32, device="cuda")
        sh["dw"] = torch.full((nw,), float("nan"), dtype=torch.float32, device="cuda")

    def stage(sh, s_):
        model.shard_backward(s_, G, B, n, p(sh, "s"), p(sh, "z1"), p(sh, "z2"), p(sh, "rot"), p(sh, "trans"),
                             p(sh, "mask"), p(sh, "dout"), k_all.data_ptr(), v_all.data_ptr(), p(sh, "dk_part"),
                             p(sh, "dv_part"), p(sh, "dk_own"), p(sh, "dv_own"), p(sh, "dt_sums"), p(sh, "ds"),
                             p(sh, "dz1"), p(sh, "dz2"), p(sh, "drot"), p(sh, "dtrans"), p(sh, "dw"), p(sh, "ws"),
                             sh["ws"].numel(), st)

    for sh in ranks:
        stage(sh, 1)
    for r, sh in enumerate(ranks):  # reduce-scatter of the partial key gradients
        sh["dk_own"].copy_(sum(o["dk_part"].view(G, -1)[r] for o in ranks))
        sh["dv_own"].copy_(sum(o["dv_part"].view(G, -1)[r] for o in ranks))
    for sh in ranks:
        stage(sh, 2)
    dt_tot = sum(sh["dt_sums"] for sh in ranks)  # all-reduce
    for sh in ranks:
        sh["dt_sums"].copy_(dt_tot)
        stage(sh, 3)
    torch.cuda.synchronize()
    out = torch.cat(outs, 1).cpu().numpy().astype(np.float64)
    assert rel_dev(ref_out, out) < 1e-3
    cat = lambda k: torch.cat([sh[k] for sh in ranks], 1).cpu().numpy().astype(np.float64)  # noqa: E731
    for k, name in (("ds", "s"), ("dz1", "z1"), ("dz2", "z2"), ("drot", "rot"), ("dtrans", "trans")):
        got = cat(k).reshape(ref_g[name].shape)
        assert np.all(np.isfinite(got)), k
        assert rel_dev(ref_g[name], got) < 5e-3, (k, rel_dev(ref_g[name], got))
    dw = sum(sh["dw"] for sh in ranks).cpu().numpy().astype(np.float64)  # all-reduce
    ref_w = np.concatenate([ref_g[nm].ravel() for nm in fo.WEIGHT_NAMES])
    assert rel_dev(ref_w, dw) < 5e-3
    if n >= 1024:
        eo, eg = emulated_backward(MAIN, oracle_weights_for(model, "bf16"), batch, dout)
        assert rel_dev(eo, out) < BF16_TOL
        for k, name in (("ds", "s"), ("dz1", "z1"), ("dz2", "z2"), ("drot", "rot"), ("dtrans", "trans")):
            assert rel_dev(eg[name], cat(k).reshape(eg[name].shape)) < BF16_TOL, k
        o = 0
        for nm in fo.WEIGHT_NAMES:
            size = eg[nm].size
            assert rel_dev(eg[nm].ravel(), dw[o:o + size]) < BF16_TOL, nm
            o += size


def test_nccl_world1_sharded_training_equals_training(fipa):
    from helpers import gpu_train_device

    model = fipa.Model(**MAIN, precision="bf16", seed=2, enforce_head_cap=False)
    B, L = 1, 256
    batch = make_batch(MAIN, B, L, seed=8, mask_frac=0.1, bf16=True)
    dout = np.random.default_rng(1).standard_normal((B, L, MAIN["d_in"]))
    ref_out, ref_g, _, _ = gpu_train_device(model, batch, dout)
    t = _dev(batch)
    dt = torch.from_numpy(dout.astype(np.float32)).cuda()
    comm = fipa.Comm(1, 0, fipa.comm_unique_id(), 0)
    nb = model.sharded_train_workspace_size(B, L, 1)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    out = torch.empty((B, L, MAIN["d_in"]), dtype=torch.float32, device="cuda")
    g = {k: torch.full_like(t[k], float("nan")) for k in ("s", "z1", "z2", "rot", "trans")}
    gw = torch.full((model.num_weights(),), float("nan"), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    args = [t[k].data_ptr() for k in ("s", "z1", "z2", "rot", "trans")] + [t["mask"].data_ptr()]
    model.forward_train_sharded_device(comm, B, L, *args, out.data_ptr(), ws.data_ptr(), nb, st)
    model.backward_sharded_device(comm, B, L, *args, dt.data_ptr(), g["s"].data_ptr(), g["z1"].data_ptr(),
                                  g["z2"].data_ptr(), g["rot"].data_ptr(), g["trans"].data_ptr(), gw.data_ptr(),
                                  ws.data_ptr(), nb, st)
    torch.cuda.synchronize()
    assert rel_dev(ref_out, out.cpu().numpy().astype(np.float64)) < 1e-3
    for k in ("s", "z1", "z2", "rot", "trans"):
        assert rel_dev(ref_g[k], g[k].cpu().numpy().astype(np.float64).reshape(ref_g[k].shape)) < 5e-3, k
    ref_w = np.concatenate([ref_g[nm].ravel() for nm in fo.WEIGHT_NAMES])
    assert rel_dev(ref_w, gw.cpu().numpy().astype(np.float64)) < 5e-3
