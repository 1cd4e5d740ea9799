"""Data-parallel plumbing: one process per GPU, pixels sharded by view, the
gradient averaged by the library's NCCL all-reduce.  torch.distributed is used only to
broadcast the 128-byte NCCL unique id and for barriers."""
from __future__ import annotations

from . import synth


def broadcast_unique_id(make_id, rank: int, world: int) -> bytes:
    """Rank 0 creates the id with make_id(); every rank returns the same 128 bytes."""
    uid = make_id() if rank == 0 else None
    if world > 1:
        import torch.distributed as dist

        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def init_comm(ctx, rank: int, world: int):
    """NCCL communicator of the library context (dinr_nccl_unique_id + dinr_comm_init)."""
    from . import _lib

    uid = broadcast_unique_id(_lib.nccl_unique_id, rank, world)
    _lib.comm_init(ctx, uid, rank, world)
    return uid


def shard_batch(name: str, n: int, rank: int, world: int, seed: int = 3, **over):
    """This rank's |Omega_k| = n pixel indices: views k with k % world == rank."""
    return synth.pixel_batch(name, n, seed=seed, rank=rank, world=world, **over)
