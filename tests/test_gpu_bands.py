"""Multi-GPU band path emulated on one GPU: every rank's omniseg_segment_band runs on the
same GPU, with the global pad colour and Otsu histogram that the NCCL collectives would
deliver injected (omniseg_debug_band_globals). Owned canvas rows must be BIT-IDENTICAL
to the single-GPU omniseg_segment_slide run (fixed-point stitch, R12), kept
tiles must be exactly the full-slide tiles that intersect the band, and the band areas
must sum to the full areas."""
import numpy as np
import pytest

from omniseg_inputs import arch_dict, arch_string, make_slide, make_weights

pytestmark = pytest.mark.gpu

H, W, PAD, P, S = 3072, 1024, 128, 256, 128
SCALES, CLASSES = (1, 2, 4), (0, 1, 1)


@pytest.fixture(scope="module")
def setup(gpu_lib):
    from paper_2305_14566_b200 import Omniseg
    a = arch_dict(levels=3, base=8, ncls=2, scale_codes=(1, 2, 4), slide_mag=4, batch=16)
    blob = make_weights(a, 1)
    spec = dict(kind="blobs", seed=31, W=W, H=H, n_blobs=14, axes=(60, 260), rings=True, nuclei=True)
    slide = make_slide(spec).numpy()
    h = Omniseg(arch_string(a), blob)
    n = sum(h.output_size(H, W, s) for s in SCALES)
    prob = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    area = np.zeros(len(SCALES), np.uint64)
    h.segment_slide(slide, H, W, PAD, P, S, SCALES, CLASSES, prob, mask, area)
    pc, hist = h.detection()
    return a, blob, slide, h, prob, mask, area, pc, hist, h.tiles()


def _split(arr, a):
    out, o = [], 0
    for s in SCALES:
        f = a["slide_mag"] // s
        hh, ww = (H + f - 1) // f, (W + f - 1) // f
        out.append(arr[o:o + hh * ww].reshape(hh, ww))
        o += hh * ww
    return out


def _window_rows(v, Hp):
    f = 1 << (v >> 30)
    oy = min(((v >> 15) & 0x7FFF) * S, Hp // f - P)
    return oy * f, (oy + P) * f


@pytest.mark.parametrize("world", [2, 3, 8])
def test_bands_bit_exact(setup, world):
    from paper_2305_14566_b200 import Omniseg
    from paper_2305_14566_b200 import dist as D
    a, blob, slide, h_full, prob, mask, area, pc, hist, tiles_full = setup
    Hp, _ = D.padded_extent(H, W, PAD)
    fmax = max(a["slide_mag"] // s for s in SCALES)
    P_full, M_full = _split(prob, a), _split(mask, a)
    area_sum = np.zeros(len(SCALES), np.uint64)
    h = Omniseg(arch_string(a), blob)
    h.band_globals(pc, hist)
    for (row0, row1) in D.band_partition(Hp, world, S):
        b0, b1 = D.band_slide_rows(H, PAD, P, fmax, row0, row1)
        own = [D.owned_canvas_rows(H, PAD, a["slide_mag"] // s, row0, row1) for s in SCALES]
        n = sum((r1 - r0) * ((W + f - 1) // f) for (r0, r1), f in zip(own, [a["slide_mag"] // s for s in SCALES]))
        bp = np.zeros(max(n, 1), np.float32)
        bm = np.zeros(max(n, 1), np.uint8)
        ba = np.zeros(len(SCALES), np.uint64)
        h.segment_band(np.ascontiguousarray(slide[b0:b1]), H, W, row0, row1, PAD, P, S, SCALES, CLASSES, bp, bm, ba)
        o = 0
        for t, ((r0, r1), s) in enumerate(zip(own, SCALES)):
            f = a["slide_mag"] // s
            ww = (W + f - 1) // f
            got_p = bp[o:o + (r1 - r0) * ww].reshape(r1 - r0, ww)
            got_m = bm[o:o + (r1 - r0) * ww].reshape(r1 - r0, ww)
            assert (got_p.view(np.uint32) == P_full[t][r0:r1].view(np.uint32)).all(), (row0, t)
            assert (got_m == M_full[t][r0:r1]).all()
            o += (r1 - r0) * ww
        area_sum += ba
        band_tiles = set(h.tiles().tolist())
        expect = {v for v in tiles_full.tolist() if _window_rows(v, Hp)[0] < row1 and _window_rows(v, Hp)[1] > row0}
        assert band_tiles == expect
        _, t_band, gp_band = h.fgmask()
    assert (area_sum == area).all()


def test_nccl_plumbing_world1(setup):
    """The real NCCL path (dlopen'ed libnccl, communicator from a torch-generated unique id,
    pad-colour broadcast, histogram and area all-reduces) with a communicator of size 1:
    the single band [0, Hp) must reproduce segment_slide bit for bit; then the NCCL band
    gather (ncclSend/ncclRecv group, the root's band as a self pair) assembles the
    full-slide device outputs on rank 0, bit-identical to segment_slide's."""
    import torch
    from paper_2305_14566_b200 import Omniseg
    from paper_2305_14566_b200 import dist as D
    a, blob, slide, h_full, prob, mask, area, pc, hist, tiles_full = setup
    h = Omniseg(arch_string(a), blob)
    h.comm_init(torch.cuda.nccl.unique_id(), 1, 0)
    Hp, _ = D.padded_extent(H, W, PAD)
    bp = np.zeros_like(prob)
    bm = np.zeros_like(mask)
    ba = np.zeros_like(area)
    with pytest.raises(Exception, match="multiples of 8"):   # argument error agreed on, then raised
        h.segment_band(slide, H, W, S, Hp, PAD, P, S, SCALES, CLASSES, bp, bm, ba)
    h.segment_band(slide, H, W, 0, Hp, PAD, P, S, SCALES, CLASSES, bp, bm, ba)
    assert (bp.view(np.uint32) == prob.view(np.uint32)).all() and (bm == mask).all() and (ba == area).all()
    # device-resident band outputs -> gather to rank 0
    dbp = torch.empty(prob.size, dtype=torch.float32, device="cuda")
    dbm = torch.empty(mask.size, dtype=torch.uint8, device="cuda")
    h.segment_band(torch.from_numpy(slide).cuda(), H, W, 0, Hp, PAD, P, S, SCALES, CLASSES, dbp, dbm, None)
    fp = torch.full((prob.size,), -1.0, dtype=torch.float32, device="cuda")
    fm = torch.full((mask.size,), 7, dtype=torch.uint8, device="cuda")
    h.gather_bands(0, H, W, PAD, D.band_cuts(Hp, 1, S), SCALES, dbp, dbm, fp, fm)
    torch.cuda.synchronize()
    assert (fp.cpu().numpy().view(np.uint32) == prob.view(np.uint32)).all()
    assert (fm.cpu().numpy() == mask).all()
    with pytest.raises(Exception, match="device"):
        h.gather_bands(0, H, W, PAD, D.band_cuts(Hp, 1, S), SCALES, bp, bm, fp, fm)   # host band buffers
    with pytest.raises(Exception, match="root needs device"):   # host outputs on the root
        h.gather_bands(0, H, W, PAD, D.band_cuts(Hp, 1, S), SCALES, dbp, dbm, np.zeros_like(prob), fm)
    # the argument agreement leaves the communicator usable: a correct gather still works
    fp.fill_(-1.0)
    h.gather_bands(0, H, W, PAD, D.band_cuts(Hp, 1, S), SCALES, dbp, dbm, fp, fm)
    torch.cuda.synchronize()
    assert (fp.cpu().numpy().view(np.uint32) == prob.view(np.uint32)).all()


def test_empty_band_joins_without_compute(setup):
    """More ranks than row units (dist.band_cuts gives them (Hp, Hp)): segment_band computes
    nothing, returns the (injected, i.e. all-reduced) global areas = 0 contribution, no tiles."""
    from paper_2305_14566_b200 import Omniseg
    from paper_2305_14566_b200 import dist as D
    a, blob, slide, h_full, prob, mask, area, pc, hist, tiles_full = setup
    Hp, _ = D.padded_extent(H, W, PAD)
    cuts = D.band_cuts(Hp, 64, S)
    assert cuts[0] == 0 and cuts[1] > 0 and cuts[-2] == Hp and cuts[-1] == Hp
    h = Omniseg(arch_string(a), blob)
    h.band_globals(pc, hist)
    ba = np.ones(len(SCALES), np.uint64)
    h.segment_band(None, H, W, Hp, Hp, PAD, P, S, SCALES, CLASSES, None, None, ba)
    assert (ba == 0).all() and len(h.tiles()) == 0
    _, t, gp = h.fgmask()
    assert t == h_full.fgmask()[1]


def test_bands_component_removal_bit_exact(setup):
    """SURVEY N2 on the band path (arch fgmin): the bands exchange their owned level-8
    foreground rows (emulated here by injecting the whole slide's pre-filter foreground, as the
    NCCL all-reduce delivers it), label the whole grid, and their owned canvas rows must be
    bit-identical to the single-GPU fgmin run; the kept windows follow the filtered mask."""
    import scipy.ndimage as ndi
    from paper_2305_14566_b200 import Omniseg
    from paper_2305_14566_b200 import dist as D
    a, blob, slide, h_full, prob, mask, area, pc, hist, tiles_full = setup
    fg_pre, _, _ = h_full.fgmask()
    lab, n = ndi.label(fg_pre, structure=[[0, 1, 0], [1, 1, 1], [0, 1, 0]])
    sizes = np.sort(np.bincount(lab.ravel())[1:])
    assert n >= 3
    fgmin = int(sizes[len(sizes) // 2]) + 1          # drops about half of the components
    af = dict(a, fgmin=fgmin)
    hf = Omniseg(arch_string(af), blob)
    nout = prob.size
    fprob = np.zeros(nout, np.float32)
    fmask = np.zeros(nout, np.uint8)
    farea = np.zeros(len(SCALES), np.uint64)
    hf.segment_slide(slide, H, W, PAD, P, S, SCALES, CLASSES, fprob, fmask, farea)
    fg_post, _, _ = hf.fgmask()
    assert fg_post.sum() < fg_pre.sum()
    Hp, _ = D.padded_extent(H, W, PAD)
    fmax = max(a["slide_mag"] // s for s in SCALES)
    Pf, Mf = _split(fprob, a), _split(fmask, a)
    hb = Omniseg(arch_string(af), blob)
    hb.band_globals(pc, hist)
    hb.band_fg(fg_pre)
    area_sum = np.zeros_like(farea)
    for (row0, row1) in D.band_partition(Hp, 3, S):
        b0, b1 = D.band_slide_rows(H, PAD, P, fmax, row0, row1)
        own = [D.owned_canvas_rows(H, PAD, a["slide_mag"] // s, row0, row1) for s in SCALES]
        nb = sum((r1 - r0) * ((W + f - 1) // f) for (r0, r1), f in zip(own, [a["slide_mag"] // s for s in SCALES]))
        bp = np.zeros(max(nb, 1), np.float32)
        bm = np.zeros(max(nb, 1), np.uint8)
        ba = np.zeros(len(SCALES), np.uint64)
        hb.segment_band(np.ascontiguousarray(slide[b0:b1]), H, W, row0, row1, PAD, P, S, SCALES, CLASSES, bp, bm, ba)
        assert (hb.fgmask()[0] == fg_post).all()
        o = 0
        for t, ((r0, r1), s) in enumerate(zip(own, SCALES)):
            f = a["slide_mag"] // s
            ww = (W + f - 1) // f
            assert (bp[o:o + (r1 - r0) * ww].view(np.uint32) == Pf[t][r0:r1].ravel().view(np.uint32)).all(), (row0, t)
            assert (bm[o:o + (r1 - r0) * ww] == Mf[t][r0:r1].ravel()).all()
            o += (r1 - r0) * ww
        area_sum += ba
    assert (area_sum == farea).all()
