"""Expert parallelism (EP) over one NVSwitch box: one process per GPU, the
M experts sharded in contiguous ranges (rank r owns partition(M, G)[r]).

Router, coreset and re-route run replicated on every rank (deterministic, so
all ranks derive the same route without communicating). Each rank streams only
its experts; its FFN epilogues push the gate-scaled slot rows into every
rank's slot buffer over NVLink peer memory and signal each rank's arrival
counter; each rank's combine waits for all arrivals and sums every token's
slots in ascending expert order — bit-identical to one GPU (C ABI:
desmoe_experts_create_ep / desmoe_ep_export / desmoe_ep_import,
include/desmoe.h). The only host-side exchange is the one-time all-gather of
128-byte IPC handles at setup.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

from . import _lib
from ._lib import check, lib


def partition(experts: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced expert ranges [lo, hi) per rank (rank order)."""
    if world < 1 or world > 8:
        raise ValueError("world outside [1, 8]")
    if experts < world:
        raise ValueError("fewer experts than ranks")
    return [((experts * r) // world, (experts * (r + 1)) // world) for r in range(world)]


def owner_of(expert: int, experts: int, world: int) -> int:
    """Rank owning `expert` under partition()."""
    for r, (lo, hi) in enumerate(partition(experts, world)):
        if lo <= expert < hi:
            return r
    raise ValueError("expert out of range")


def export_handle(ex) -> bytes:
    """This rank's 128-byte IPC handle blob (slot buffer + arrival counter)."""
    buf = (C.c_ubyte * _lib.EP_HANDLE_BYTES)()
    check(lib().desmoe_ep_export(ex.h, buf))
    return bytes(buf)


def all_gather_handles(blob: bytes, group=None) -> bytes:
    """All-gather every rank's handle blob in rank order over torch.distributed
    (gloo on CPU tensors, or nccl on CUDA tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    mine = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return b"".join(bytes(p.cpu().numpy().tobytes()) for p in parts)


def import_handles(ex, world: int, rank: int, blobs: bytes) -> None:
    if len(blobs) != world * _lib.EP_HANDLE_BYTES:
        raise ValueError("handle blob size does not match world")
    buf = (C.c_ubyte * len(blobs)).from_buffer_copy(blobs)
    check(lib().desmoe_ep_import(ex.h, world, rank, buf))


def connect_distributed(ex, group=None) -> None:
    """Wire this rank's experts to its peers (collective over `group`)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    blobs = all_gather_handles(export_handle(ex), group)
    import_handles(ex, world, rank, blobs)


def connect_local(experts: Sequence) -> None:
    """Wire G expert shards living in ONE process (same device or peer-capable
    devices) — the single-GPU EP simulation the tests use."""
    world = len(experts)
    slots = (C.c_void_p * world)()
    flags = (C.c_void_p * world)()
    for r, ex in enumerate(experts):
        sp, fp = C.c_void_p(), C.c_void_p()
        sb, fb = C.c_size_t(), C.c_size_t()
        check(lib().desmoe_ep_local_buffers(ex.h, C.byref(sp), C.byref(sb), C.byref(fp),
                                            C.byref(fb)))
        slots[r], flags[r] = sp.value, fp.value
    for r, ex in enumerate(experts):
        check(lib().desmoe_ep_connect(ex.h, world, r, slots, flags))
