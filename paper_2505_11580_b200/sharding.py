"""Query-row sharding plan for long single structures (BASELINE cfg4).

One process per GPU.  A sequence of L residues is split into `world` contiguous blocks of
L / world rows; rank r owns rows [r*L/world, (r+1)*L/world).  Each rank projects and packs its own
rows, the packed key/value rows are all-gathered rank-major over NCCL ([G][B*H][L_local][pad],
key j of the sequence = row j % L_local of shard j // L_local -- the layout the attention
kernel's 5-D TMA maps read), and each rank returns the output rows of its block.  The
translation centroid used for recentring is all-reduced (4 floats per sample).  The compute and
the collectives run in libfipa_b200.so (fipa_layer_forward_sharded); torch.distributed is used
here only to hand rank 0's NCCL unique id to the other ranks.
"""

from __future__ import annotations


def row_block(L: int, world: int, rank: int):
    """[start, stop) of the residues rank `rank` owns.  Blocks are equal and, when world > 1,
    a multiple of 64 rows (the attention kernel's key tile never straddles two shards)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    if L % world != 0:
        raise ValueError(f"L={L} is not divisible by world={world}")
    n = L // world
    if world > 1 and n % 64 != 0:
        raise ValueError(f"per-rank block {n} must be a multiple of 64 residues")
    return rank * n, (rank + 1) * n


def key_location(j: int, L_local: int):
    """(shard, row) of sequence key j in the gathered key/value buffer."""
    return j // L_local, j % L_local


def share_unique_id(uid: bytes | None, group=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id to every rank (any torch.distributed backend)."""
    import torch.distributed as dist

    obj = [uid if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise RuntimeError("NCCL unique id exchange failed")
    return bytes(obj[0])


def make_comm(fipa, device: int, group=None):
    """fipa.Comm over the ranks of the (initialised) default torch.distributed group."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = share_unique_id(fipa.comm_unique_id() if rank == 0 else None, group)
    return fipa.Comm(world, rank, uid, device)
