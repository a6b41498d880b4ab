"""GPU parity at every level factor f = 1, 2, 4, 8 (40x / 20x / 10x / 5x tasks in ONE call),
element-wise over whole canvases (VERDICT r1 'What's missing' #2; §2.2 "tiled into
small regions at three different scales (40x, 10x, and 5x)"):

* probe network (tests/special_nets.py): canvas = sigmoid(G_f / 256 - 11/16) of the level
  image wherever a kept window covers -- a closed form that pins the L2 / L4 / L8 pyramid
  levels the fused gather + stem reads and the canvas placement `oy - pad / f` of every
  scale; |dp| <= 2e-6 (fp32 sigmoid + 2^-20 fixed point), masks exact except within 2e-6 of 1/2;
* shift-identity network: the whole trunk's spatial bookkeeping at every scale, through the
  bench network's kernels (levels 5, base 32), against its closed form, |dp| <= 2e-6;
* random networks (the tiny config-1 net and the config-2+ bench net at 256^2 windows) against
  the fp64 oracle: the north_star gates (|dp| <= 1e-2, masks >= 99.9 % with every flip
  within 1e-2 of 1/2), tile lists and foreground bit-exact.
"""
import numpy as np
import pytest

from omniseg_inputs import arch_string, make_slide, workload
from omniseg_inputs.arch import arch_dict, make_weights
from oracle import frontend as fe
from oracle import pipeline as op

from special_nets import block_mean_brute, head_theta, probe_net, shift_identity_F, shift_identity_net

pytestmark = pytest.mark.gpu

SCALES = (40, 20, 10, 5)          # f = 1, 2, 4, 8
CLASSES = (4, 2, 3, 0)            # PTC, PT, DT, TUFT


def _slide(crop=None):
    s = make_slide(workload(1).slide).numpy()
    return s if crop is None else s[:crop[0], :crop[1]].copy()


def _unpack(ids, Hp, Wp, P, S):
    out = []
    for v in ids.tolist():
        f = 1 << (v >> 30)
        out.append((f, min(((v >> 15) & 0x7FFF) * S, Hp // f - P), min((v & 0x7FFF) * S, Wp // f - P)))
    return out


def _run(a, blob, slide, pad, P, S, scales=SCALES, classes=CLASSES):
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(a), blob)
    H, W = slide.shape[:2]
    sizes = [h.output_size(H, W, s) for s in scales]
    prob = np.zeros(sum(sizes), np.float32)
    mask = np.zeros(sum(sizes), np.uint8)
    area = np.zeros(len(scales), np.uint64)
    h.segment_slide(slide, H, W, pad, P, S, scales, classes, prob, mask, area)
    out, o = [], 0
    for s, n in zip(scales, sizes):
        f = 40 // s
        shp = ((H + f - 1) // f, (W + f - 1) // f)
        out.append((prob[o:o + n].reshape(shp), mask[o:o + n].reshape(shp)))
        o += n
    return h, out, area


def _kept(slide, pad, P, S, factors):
    fr = op.front_end(slide, pad, P, S, factors)
    return fr, fr["kept"]


def _canvas_from_windows(kept, f, pad, P, Ht, Wt, pfun):
    """Mean over covering kept windows of scale f of the per-window map pfun(k) (closed forms)."""
    acc = np.zeros((Ht, Wt))
    cnt = np.zeros((Ht, Wt), np.int64)
    for k in kept:
        if k[0] != f:
            continue
        oy, ox = k[1] - pad // f, k[2] - pad // f
        a0, a1, b0, b1 = max(0, oy), min(Ht, oy + P), max(0, ox), min(Wt, ox + P)
        if a0 >= a1 or b0 >= b1:
            continue
        acc[a0:a1, b0:b1] += pfun(k)[a0 - oy:a1 - oy, b0 - ox:b1 - ox]
        cnt[a0:a1, b0:b1] += 1
    return np.where(cnt > 0, acc / np.maximum(cnt, 1), 0.0), cnt


@pytest.mark.parametrize("levels, base, P, S, pad, crop", [
    (3, 8, 64, 32, 64, (520, 392)),          # tiny net, ragged slide
    (5, 32, 256, 128, 512, None),            # bench network's kernels, 1024^2 slide in a 2048^2 frame
])
def test_probe_network_all_scales_closed_form(gpu_lib, levels, base, P, S, pad, crop):
    slide = _slide(crop)
    H, W = slide.shape[:2]
    theta = head_theta(1.0 / 256, -0.6875, ch=1)
    a, net, blob = probe_net(levels, base, theta, ncls=6, scale_codes=(5, 10, 20, 40), slide_mag=40)
    h, out, area = _run(a, blob, slide, pad, P, S)
    fr, kept = _kept(slide, pad, P, S, [8, 4, 2, 1])
    assert _unpack(h.tiles(), fr["Hp"], fr["Wp"], P, S) == kept
    for t, s in enumerate(SCALES):
        f = 40 // s
        Ht, Wt = (H + f - 1) // f, (W + f - 1) // f
        Lf = block_mean_brute(fr["padded"], f)
        G = Lf[pad // f:pad // f + Ht, pad // f:pad // f + Wt, 1].astype(np.float64)
        exp = 1.0 / (1.0 + np.exp(-(G / 256 - 0.6875)))
        _, cnt = _canvas_from_windows(kept, f, pad, P, Ht, Wt, lambda k: np.zeros((P, P)))
        cov = cnt > 0
        p, m = out[t]
        assert cov.any(), f
        d = np.abs(p.astype(np.float64) - np.where(cov, exp, 0.0))
        assert d.max() <= 2e-6, (f, d.max())
        dis = m != (cov & (exp >= 0.5))
        assert (np.abs(exp[dis] - 0.5) <= 2e-6).all(), f
        assert int(area[t]) == int(m.sum())
        assert 0 < m[cov].mean() < 1, f
        print(f"probe f={f}: {int(cov.sum())} covered px, max |dp| {d.max():.2e}")


@pytest.mark.parametrize("levels, base, P, S, pad", [(3, 8, 128, 64, 128), (5, 32, 256, 128, 512)])
def test_shift_identity_network_all_scales(gpu_lib, levels, base, P, S, pad):
    """z = F_0 / 256 - 2 with F the shift-identity trunk: every window's map is a closed form of
    its level window, so the stitched canvas of every scale is the mean of closed forms."""
    slide = _slide()
    H, W = slide.shape[:2]
    theta = head_theta(1.0 / 256, -2.0)
    a, net, blob = shift_identity_net(levels, base, bc=theta, ncls=6, scale_codes=(5, 10, 20, 40), slide_mag=40)
    h, out, area = _run(a, blob, slide, pad, P, S)
    fr, kept = _kept(slide, pad, P, S, [8, 4, 2, 1])
    assert _unpack(h.tiles(), fr["Hp"], fr["Wp"], P, S) == kept
    pc = fe.pad_colour(slide)
    for t, s in enumerate(SCALES):
        f = 40 // s
        Ht, Wt = (H + f - 1) // f, (W + f - 1) // f

        def pfun(k):
            win = fe.level_window(slide, pad, pc, f, k[1], k[2], P)
            return 1.0 / (1.0 + np.exp(-(shift_identity_F(win, levels)[:, :, 0] / 256 - 2.0)))

        ref, cnt = _canvas_from_windows(kept, f, pad, P, Ht, Wt, pfun)
        p, m = out[t]
        d = np.abs(p.astype(np.float64) - ref)
        assert d.max() <= 2e-6, (f, d.max())
        dis = m != ((cnt > 0) & (ref >= 0.5))
        assert (np.abs(ref[dis] - 0.5) <= 2e-6).all(), f
        cv = ref[cnt > 0]
        assert cv.std() > 1e-3, f                      # informative (f = 8: one mostly-background window)
        print(f"shift-identity f={f}: {int((cnt > 0).sum())} covered px, max |dp| {d.max():.2e}")


def _gates(p_gpu, m_gpu, p_ref, m_ref, tag):
    d = np.abs(p_gpu.astype(np.float64) - p_ref)
    assert d.max() <= 1e-2, f"{tag}: max |dp| {d.max():.4g}"
    dis = m_gpu != m_ref
    assert 1.0 - dis.mean() >= 0.999, f"{tag}: mask agreement {1 - dis.mean():.5f}"
    assert (np.abs(p_ref[dis] - 0.5) <= 1e-2).all(), f"{tag}: mask flip away from 1/2"
    return d.max(), 1.0 - dis.mean()


def _random_net_case(a, blob, slide, pad, P, S):
    ref = op.segment_slide(slide, blob, arch_string(a), pad, P, S, SCALES, CLASSES)
    h, out, area = _run(a, blob, slide, pad, P, S)
    fr_hp, fr_wp = fe.padded_extent(slide.shape[0], slide.shape[1], pad)
    assert _unpack(h.tiles(), fr_hp, fr_wp, P, S) == ref["kept"]
    fg, t, gpad = h.fgmask()
    assert t == ref["t"] and (fg == ref["fg"]).all()
    for i, s in enumerate(SCALES):
        f = 40 // s
        dmax, agree = _gates(out[i][0], out[i][1], ref["prob"][i], ref["mask"][i], f"f={f}")
        assert int(area[i]) == int(out[i][1].sum())
        nk = sum(1 for k in ref["kept"] if k[0] == f)
        assert nk > 0 and (ref["cnt"][i] > 0).any()
        print(f"f={f}: {nk} windows, max |dp| {dmax:.3g}, mask agreement {agree:.6f}")


def test_tiny_net_all_scales_elementwise(gpu_lib):
    """Config-1 network (3 levels, base 8, random He weights) at 4 scales, 128^2 windows."""
    a = arch_dict(levels=3, base=8, ncls=6, scale_codes=(5, 10, 20, 40), slide_mag=40, batch=16)
    _random_net_case(a, make_weights(a, 1), _slide(), 128, 128, 64)


@pytest.mark.slow
def test_bench_net_all_scales_elementwise(gpu_lib):
    """The config-2+ bench network (5 levels, base 32, calibrated head, fp16f8, batch 64) at 4
    scales on 256^2 windows (the 1024^2 slide in a 2048^2 frame, so a 5x window fits)."""
    w = workload(3)
    _random_net_case(w.arch, w.weights(), _slide(), 512, 256, 128)
