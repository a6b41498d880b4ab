"""Multi-GPU row-band driver: one process per GPU, torch.distributed for
the plumbing, the library's own NCCL communicator for the data-path collectives.

Host logic only -- every pixel is computed by libomniseg (omniseg_segment_band).
"""
from __future__ import annotations

from . import lib


def padded_extent(H: int, W: int, pad: int):
    r = lambda v: (v + 127) // 128 * 128  # noqa: E731
    return r(H + 2 * pad), r(W + 2 * pad)


def band_cuts(Hp: int, world: int, stride: int):
    """world+1 band boundaries of the padded 40x frame: contiguous bands whose boundaries are
    multiples of 8*stride (so every scale's tile rows and the level-8 grid align), the last
    band ending at Hp; the nb = ceil(Hp / (8 stride)) row units are split as evenly as
    possible over min(world, nb) ranks -- rank 0 always holds row 0 (the pad colour, the
    broadcast root) and ranks beyond nb get EMPTY bands (Hp, Hp), which join the collectives
    without compute (omniseg.h)."""
    unit = 8 * stride
    nb = (Hp + unit - 1) // unit
    act = min(world, nb)
    cuts = [min(Hp, (nb * min(r, act) // act) * unit) for r in range(world + 1)]
    cuts[-1] = Hp
    return cuts


def band_partition(Hp: int, world: int, stride: int):
    """Owned rows [row0, row1) per rank (band_cuts)."""
    cuts = band_cuts(Hp, world, stride)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def band_halo(patch: int, fmax: int) -> int:
    """Slide rows a band needs beyond its owned rows: one window at the coarsest scale
    plus the detection median's reach (3 level-8 rows), rounded up (omniseg.h)."""
    return patch * fmax + 64


def band_slide_rows(H: int, pad: int, patch: int, fmax: int, row0: int, row1: int):
    """Slide rows [b0, b1) the caller passes as rgb_band for the band [row0, row1)."""
    halo = band_halo(patch, fmax)
    b0 = max(0, min(H, row0 - pad - halo))
    b1 = max(0, min(H, row1 - pad + halo))
    return b0, b1


def owned_canvas_rows(H: int, pad: int, f: int, row0: int, row1: int):
    """Owned rows of a task canvas at level factor f (omniseg_band_rows)."""
    return lib.band_rows(H, row0, row1, pad, f)


def init_comm(h, world: int, rank: int):
    """Create the library's NCCL communicator: rank 0's unique id is broadcast through
    torch.distributed (any backend)."""
    if world <= 1:
        return
    import torch
    import torch.distributed as dist
    uid = torch.cuda.nccl.unique_id() if rank == 0 else None
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    h.comm_init(obj[0], world, rank)
