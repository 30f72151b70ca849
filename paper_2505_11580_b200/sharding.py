"""Query-row sharding plan for long single structures (BASELINE cfg4).

One process per GPU.  A sequence of L residues is split into `world` contiguous blocks of
L / world rows; rank r owns rows [r*L/world, (r+1)*L/world).  Each rank projects and packs its own
rows, the packed key/value rows are all-gathered rank-major over NCCL ([G][B*H][L_local][pad],
key j of the sequence = row j % L_local of shard j // L_local -- the layout the attention
kernel's 5-D TMA maps read), and each rank returns the output rows of its block.  The
translation centroid used for recentring is all-reduced (4 floats per sample).  The compute and
the collectives run in libfipa_b200.so (fipa_layer_forward_sharded).  The only host-side exchange
is rank 0's 128-byte NCCL unique id: any byte-broadcast callable can carry it (MPI, a key-value
store, a file); torch.distributed is used only when no callable is given.
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


def share_unique_id(uid: bytes | None, group=None, broadcast=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id to every rank.

    broadcast: optional callable(bytes | None) -> bytes that returns rank 0's payload on every
    rank (rank 0 passes the id, the others None).  Without it, torch.distributed (any backend,
    `group` or the default group) carries it."""
    if broadcast is not None:
        got = broadcast(uid)
    else:
        import torch.distributed as dist

        obj = [uid if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        got = obj[0]
    if not isinstance(got, (bytes, bytearray)) or len(got) != 128:
        raise RuntimeError("NCCL unique id exchange failed")
    return bytes(got)


def make_comm(fipa, device: int, group=None, *, world: int | None = None, rank: int | None = None,
              broadcast=None):
    """fipa.Comm over `world` ranks.  With `broadcast` (see share_unique_id) the caller names world
    and rank itself and torch is not needed; otherwise they come from the (initialised)
    torch.distributed group."""
    if broadcast is None:
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
    elif world is None or rank is None:
        raise ValueError("make_comm(broadcast=...) needs world and rank")
    uid = share_unique_id(fipa.comm_unique_id() if rank == 0 else None, group, broadcast)
    return fipa.Comm(world, rank, uid, device)
