"""CPU (gloo, world_size 2): the query-row sharding plan.  Each rank packs its own residue block
(float64 layout emulation of pack.cu), the centroid sums are all-reduced, the packed key/value
rows are all-gathered rank-major, and attention over the gathered buffer -- addressed with the
kernel's shard/row index math -- must reproduce the unsharded layer exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_11580_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import bwd_emulation as be
    from oracle import fipa_oracle as fo

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = dict(d_in=16, d_z=4, heads=2, c=8, n_query=2, n_value=3, rank=2)
        cfg = fo.IpaConfig(**shape, enforce_head_cap=False)
        w = fo.init_weights(cfg, 2)
        L = 128 * world
        p = fo.make_problem(cfg, L, 9, translation_scale=5.0, mask_frac=0.1)
        lo, hi = sharding.row_block(L, world, rank)
        # 1. centroid: local sums, all-reduced
        m = p.mask[lo:hi]
        sums = torch.tensor(np.concatenate([p.trans[lo:hi][m].sum(0), [m.sum()]]), dtype=torch.float64)
        dist.all_reduce(sums)
        cen = (sums[:3] / sums[3]).numpy()
        # 2. local pack (rows lo..hi), 3. rank-major all-gather of the packed keys / values
        pk = be.pack(cfg, w, p.s[lo:hi], p.z1[lo:hi], p.z2[lo:hi], p.rot[lo:hi], p.trans[lo:hi] - cen, p.mask[lo:hi])
        k_all = [torch.zeros_like(torch.from_numpy(pk["k_hat"])) for _ in range(world)]
        v_all = [torch.zeros_like(torch.from_numpy(pk["v_hat"])) for _ in range(world)]
        dist.all_gather(k_all, torch.from_numpy(pk["k_hat"]))
        dist.all_gather(v_all, torch.from_numpy(pk["v_hat"]))
        k_all = torch.stack(k_all).numpy()  # [G][H][L_local][d]
        v_all = torch.stack(v_all).numpy()
        n = hi - lo
        keys = [sharding.key_location(j, n) for j in range(L)]
        K = np.stack([k_all[g][:, r] for g, r in keys], 1)  # [H][L][d] in sequence order
        V = np.stack([v_all[g][:, r] for g, r in keys], 1)
        o, _ = be.attention(pk["q_hat"], K, V, L)
        feat, _ = be.epilogue(cfg, o, p.z1[lo:hi], p.rot[lo:hi], p.trans[lo:hi] - cen)
        out = feat @ w["w_out"] + w["b_out"]
        out[~p.mask[lo:hi]] = 0.0
        # unsharded reference for the same rows
        full_c = p.trans[p.mask].mean(0)
        pkf = be.pack(cfg, w, p.s, p.z1, p.z2, p.rot, p.trans - full_c, p.mask)
        of, _ = be.attention(pkf["q_hat"], pkf["k_hat"], pkf["v_hat"], L)
        ff, _ = be.epilogue(cfg, of, p.z1, p.rot, p.trans - full_c)
        ref = ff @ w["w_out"] + w["b_out"]
        ref[~p.mask] = 0.0
        q.put((rank, float(np.abs(ref[lo:hi] - out).max() / np.abs(ref).max()),
               float(np.abs(fo.flash_ipa_forward(p.s, p.z1, p.z2, p.rot, p.trans, p.mask, cfg, w)[lo:hi]
                            - out).max() / np.abs(ref).max())))
        # the NCCL unique id handed from rank 0 reaches every rank unchanged
        uid = sharding.share_unique_id(bytes(range(128)) if rank == 0 else None)
        assert uid == bytes(range(128))
    finally:
        dist.destroy_process_group()


def test_row_blocks_partition_the_sequence():
    L, world = 1024, 4
    rows = [sharding.row_block(L, world, r) for r in range(world)]
    assert rows[0][0] == 0 and rows[-1][1] == L
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    with pytest.raises(ValueError):
        sharding.row_block(1000, 4, 0)  # 250 rows: not a multiple of 64
    with pytest.raises(ValueError):
        sharding.row_block(1024, 3, 0)


def test_two_rank_gloo_sharded_plan_reproduces_unsharded_layer():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    for rank, err_layout, err_oracle in res:
        assert err_layout < 1e-12, (rank, err_layout)   # same layout arithmetic, sharded vs not
        assert err_oracle < 1e-3, (rank, err_oracle)    # vs the reference restatement (hi/lo split)


def test_unique_id_exchange_without_torch():
    """share_unique_id / make_comm take any byte-broadcast callable (no torch.distributed)."""
    from paper_2505_11580_b200 import sharding

    uid = bytes(range(128))
    box = {}

    def bcast(payload):  # a 'store': rank 0 writes, the others read
        if payload is not None:
            box["id"] = payload
        return box["id"]

    assert sharding.share_unique_id(uid, broadcast=bcast) == uid
    assert sharding.share_unique_id(None, broadcast=bcast) == uid
    with pytest.raises(RuntimeError):
        sharding.share_unique_id(None, broadcast=lambda p: b"short")
    with pytest.raises(ValueError):
        sharding.make_comm(None, 0, broadcast=bcast)


def test_product_imports_without_torch():
    """The product package (pybind module + libfipa_b200.so) imports in a process where
    `import torch` raises, and does not import torch on its own; torch still imports after it
    (the CUDA runtime is linked shared, libstdc++ dynamically)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import builtins, sys\n"
            "real = builtins.__import__\n"
            "def imp(n, *a, **k):\n"
            "    if n == 'torch' or n.startswith('torch.'): raise ImportError('torch blocked')\n"
            "    return real(n, *a, **k)\n"
            "builtins.__import__ = imp\n"
            "import paper_2505_11580_b200 as f\n"
            "assert 'torch' not in sys.modules\n"
            "from paper_2505_11580_b200 import sharding, report\n"
            "print(f.Model(seed=1).config['d_in'])\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "32", r.stderr
    code2 = "import sys, paper_2505_11580_b200\nassert 'torch' not in sys.modules\nimport torch\nprint('ok')\n"
    r = subprocess.run([sys.executable, "-c", code2], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr
