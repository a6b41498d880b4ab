"""World-size-2 gloo test (CPU) of the multi-GPU row-band host logic:
band partition, halo (slide rows each rank needs), tile ownership, owned canvas rows.
Each rank recomputes its band with the ORACLE (tiny network) and the gathered owned
canvases must equal the single-process oracle canvas exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from omniseg_inputs import arch_dict, arch_string, make_slide, make_weights
from oracle import net as nn
from oracle import pipeline as op

H, W, PAD, P, S = 1536, 512, 64, 128, 64


def _setup():
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    spec = dict(kind="blobs", seed=21, W=W, H=H, n_blobs=8, axes=(40, 150), rings=False, nuclei=False)
    slide = make_slide(spec).numpy()
    return a, make_weights(a, 1), slide


def _band_canvas(rank, world, a, blob, slide, fr):
    from paper_2305_14566_b200 import dist as D
    Hp, Wp = D.padded_extent(H, W, PAD)
    row0, row1 = D.band_partition(Hp, world, S)[rank]
    b0, b1 = D.band_slide_rows(H, PAD, P, 1, row0, row1)
    r0, r1 = D.owned_canvas_rows(H, PAD, 1, row0, row1)
    arch = nn.parse_arch(arch_string(a))
    net = nn.unpack_weights(arch, blob)
    mine = [t for t in fr["kept"] if t[1] < row1 and t[1] + P > row0]
    # halo adequacy: every window of my tiles lies in the slide rows I hold (or in padding)
    for (_, oy, _ox) in mine:
        lo, hi = max(0, oy - PAD), min(H, oy + P - PAD)
        assert lo >= b0 and hi <= b1, (rank, oy, b0, b1)
    s = np.zeros((r1 - r0, W))
    c = np.zeros((r1 - r0, W), np.int64)
    for (_, oy, ox) in mine:
        p = nn.predict_tile(net, arch, fr["padded"][oy:oy + P, ox:ox + P], [(0, 0)])[0]
        op.stitch_add(s, c, p, oy - PAD - r0, ox - PAD)
    return (row0, row1, r0, r1, s, c, len(mine))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, blob, slide = _setup()
        fr = op.front_end(slide, PAD, P, S, [1])
        res = _band_canvas(rank, world, a, blob, slide, fr)
        out = [None] * world
        dist.all_gather_object(out, res)
        # band gather to rank 0 over point-to-point messages (the layout omniseg_gather_bands
        # uses over NCCL: rank r's owned canvas rows [r0, r1) land at rows r0..r1 of the full canvas)
        from paper_2305_14566_b200 import dist as D
        Hp, _ = D.padded_extent(H, W, PAD)
        cuts = D.band_cuts(Hp, world, S)
        s_band = torch.from_numpy(np.ascontiguousarray(res[4]))
        if rank == 0:
            full = torch.zeros((H, W), dtype=torch.float64)
            for r in range(world):
                r0, r1 = D.owned_canvas_rows(H, PAD, 1, cuts[r], cuts[r + 1])
                if r1 <= r0:
                    continue
                if r == 0:
                    full[r0:r1] = s_band
                else:
                    buf = torch.empty((r1 - r0, W), dtype=torch.float64)
                    dist.recv(buf, src=r)
                    full[r0:r1] = buf
            res = res + (full.numpy(),)
        elif res[3] > res[2]:
            dist.send(s_band, dst=0)
        obj = [fr["kept"] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == fr["kept"]
        if rank == 0:
            q.put((out, res[7]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.slow
def test_band_decomposition_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out, full = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a, blob, slide = _setup()
    ref = op.segment_slide(slide, blob, arch_string(a), PAD, P, S, (1,), (0,))
    from paper_2305_14566_b200 import dist as D
    Hp, _ = D.padded_extent(H, W, PAD)
    # bands partition the padded frame; owned canvas rows partition the canvas
    assert out[0][0] == 0 and out[-1][1] == Hp
    assert all(out[i][1] == out[i + 1][0] for i in range(world - 1))
    assert out[0][2] == 0 and out[-1][3] == H
    assert all(out[i][3] == out[i + 1][2] for i in range(world - 1))
    s = np.concatenate([o[4] for o in out])
    c = np.concatenate([o[5] for o in out])
    prob, mask = op.finalize(s, c)
    assert (c == ref["cnt"][0]).all()
    np.testing.assert_allclose(prob, ref["prob"][0], rtol=0, atol=1e-15)
    assert (mask == ref["mask"][0]).all()
    # the gathered canvas sums on rank 0 are the concatenation of the owned bands
    assert (full == s).all()
    # boundary windows are computed by both neighbours (duplication > 0, bounded)
    assert sum(o[6] for o in out) >= len(ref["kept"])


def test_band_partition_properties():
    from paper_2305_14566_b200 import dist as D
    for Hp, S, world in [(1280, 128, 2), (64128, 256, 8), (64128, 256, 3), (20480, 256, 4), (3328, 128, 4)]:
        b = D.band_partition(Hp, world, S)
        assert b[0][0] == 0 and b[-1][1] == Hp and len(b) == world
        for (r0, r1), (s0, _s1) in zip(b, b[1:]):
            assert r1 == s0 and r0 < r1 and r0 % (8 * S) == 0
        sizes = [r1 - r0 for r0, r1 in b[:-1]]
        assert max(sizes) - min(sizes) <= 8 * S


def test_band_partition_more_ranks_than_units():
    """with world > nb = ceil(Hp / 8S) row units (cfg1 at 4 / 8 GPUs, cfg2 at 8), the
    first nb ranks get one unit each (rank 0 always holds row 0, the pad-colour broadcast root)
    and the rest get EMPTY bands (Hp, Hp) that join the collectives without compute."""
    from paper_2305_14566_b200 import dist as D
    for Hp, S, world in [(1280, 128, 4), (1280, 128, 8), (5120, 256, 8), (2048, 256, 2)]:
        nb = -(-Hp // (8 * S))
        cuts = D.band_cuts(Hp, world, S)
        b = D.band_partition(Hp, world, S)
        assert cuts[0] == 0 and cuts[-1] == Hp and all(x <= y for x, y in zip(cuts, cuts[1:]))
        nonempty = [(r0, r1) for r0, r1 in b if r1 > r0]
        assert len(nonempty) == min(world, nb) and b[0][1] > 0
        assert b[:len(nonempty)] == nonempty                     # empty bands come last
        assert all(r0 == r1 == Hp for r0, r1 in b[len(nonempty):])
        assert all(r0 % (8 * S) == 0 for r0, _ in nonempty)


def test_world1_comm_init_is_noop():
    from paper_2305_14566_b200 import dist as D

    class H:
        def comm_init(self, *a):
            raise AssertionError("must not be called for world 1")
    D.init_comm(H(), 1, 0)
