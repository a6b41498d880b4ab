"""Pins for the oracle's multi-scale bookkeeping (VERDICT r1 'parity unpinned' items):

* task_factors: the level factor of a magnification (§2.2 40x / 10x / 5x copies of the
  40x scan, §3.1 0.25 um at 40x) -- f = slide_mag / scale;
* the canvas placement of a window of scale f (segment_slide's `oy - pad // f`) at f = 1,
  2, 4, 8, through the probe network whose stitched canvas is a closed form of the level
  image: canvas[cy, cx] = sigmoid(w3 L_f[cy + pad/f, cx + pad/f, ch] + b3) wherever a kept
  window covers the pixel, 0 elsewhere (tests/special_nets.py);
* mask_by_foreground: the level-8 foreground upsampled to 40x by pixel replication and
  sampled at each canvas pixel's footprint (S:350 filter_by_foreground, §2.3);
* the shift-identity closed form of the trunk at 5 levels (the bench network's depth).
"""
import numpy as np
import pytest

from omniseg_inputs import arch_string, make_slide, workload
from oracle import frontend as fe
from oracle import net as nn
from oracle import pipeline as op

from special_nets import block_mean_brute, head_theta, probe_net, shift_identity_F, shift_identity_net


def test_task_factors_table():
    arch = dict(scale_codes=[5, 10, 20, 40], slide_mag=40)
    assert op.task_factors(arch, [5, 10, 20, 40]) == [(8, 0), (4, 1), (2, 2), (1, 3)]
    assert op.task_factors(dict(scale_codes=[5, 10, 20, 40], slide_mag=10), [10, 10]) == [(1, 1), (1, 1)]
    assert op.task_factors(dict(scale_codes=[5, 10, 20, 40], slide_mag=20), [5]) == [(4, 0)]
    for bad_arch, sc in ((arch, [7]), (dict(scale_codes=[5, 40], slide_mag=40), [10]),
                         (dict(scale_codes=[3, 40], slide_mag=48), [3]), (dict(scale_codes=[5], slide_mag=80), [5])):
        with pytest.raises(ValueError):
            op.task_factors(bad_arch, sc)


def _probe_case(pad, P, S, crop):
    slide = make_slide(workload(1).slide).numpy()[:crop[0], :crop[1]].copy()
    theta = head_theta(1.0 / 256, -0.6875, ch=1)       # z = G / 256 - 11/16 (fp32-exact): tissue < 1/2 < bg
    a, net, blob = probe_net(3, 8, theta, ncls=2, scale_codes=(5, 10, 20, 40), slide_mag=40)
    scales, classes = (40, 20, 10, 5), (0, 1, 0, 1)
    r = op.segment_slide(slide, blob, arch_string(a), pad, P, S, scales, classes)
    return slide, r, scales


@pytest.mark.parametrize("pad, P, S, crop", [(64, 64, 32, (520, 392)), (128, 64, 16, (650, 470))])
def test_canvas_placement_all_level_factors_probe_network(pad, P, S, crop):
    slide, r, scales = _probe_case(pad, P, S, crop)
    H, W = slide.shape[:2]
    padded = fe.pad_slide(slide, pad)
    assert len(r["kept"]) > 0
    for t, s in enumerate(scales):
        f = 40 // s
        Lf = block_mean_brute(padded, f)
        Ht, Wt = -(-H // f), -(-W // f)
        g = Lf[pad // f:pad // f + Ht, pad // f:pad // f + Wt, 1].astype(np.float64)
        exp = 1.0 / (1.0 + np.exp(-(g / 256 - 0.6875)))
        cov = r["cnt"][t] > 0
        # coverage = union of the kept windows of this scale, placed at (oy - pad/f, ox - pad/f)
        cov_bf = np.zeros((Ht, Wt), bool)
        for (ff, oy, ox) in r["kept"]:
            if ff == f:
                cov_bf[max(0, oy - pad // f):max(0, oy - pad // f + P), max(0, ox - pad // f):max(0, ox - pad // f + P)] = True
        assert (cov == cov_bf).all(), f
        assert cov.any(), f
        np.testing.assert_allclose(r["prob"][t][cov], exp[cov], rtol=1e-12, atol=0)
        assert (r["prob"][t][~cov] == 0).all()
        assert (r["mask"][t] == (cov & (exp >= 0.5))).all()
        m = r["mask"][t][cov]
        assert 0 < m.mean() < 1, (f, m.mean())            # informative: both classes present


def test_canvas_placement_detects_a_shifted_window():
    """The closed form is sensitive to the placement: one level pixel of offset changes it."""
    slide, r, scales = _probe_case(64, 64, 32, (520, 392))
    padded = fe.pad_slide(slide, 64)
    f = 4
    Lf = block_mean_brute(padded, f)
    H, W = slide.shape[:2]
    Ht, Wt = -(-H // f), -(-W // f)
    off = 64 // f
    good = Lf[off:off + Ht, off:off + Wt, 1]
    bad = Lf[off + 1:off + 1 + Ht, off:off + Wt, 1]
    cov = r["cnt"][scales.index(10)] > 0
    assert (good[cov] != bad[cov]).mean() > 0.3


def test_mask_by_foreground_brute_force():
    """Nearest-neighbour foreground filter: the level-8 mask replicated to 40x (each level-8
    pixel an 8x8 block of the padded frame), then each canvas pixel of a level-f task takes
    the value at its footprint (padded rows [cy f + pad, (cy+1) f + pad)), which lies inside
    one 8x8 block for f in {1, 2, 4, 8} and pad % 8 == 0."""
    rng = np.random.default_rng(4)
    pad = 24
    H, W = 77, 101
    Hp, Wp = fe.padded_extent(H, W, pad)
    fg8 = (rng.random((Hp // 8, Wp // 8)) < 0.5).astype(np.uint8)
    fg40 = np.kron(fg8, np.ones((8, 8), np.uint8))
    for f in (1, 2, 4, 8):
        Ht, Wt = -(-H // f), -(-W // f)
        mask = (rng.random((Ht, Wt)) < 0.7).astype(np.uint8)
        got = op.mask_by_foreground(mask, fg8, f, pad)
        exp = np.zeros_like(mask)
        for cy in range(Ht):
            for cx in range(Wt):
                blk = fg40[cy * f + pad:(cy + 1) * f + pad, cx * f + pad:(cx + 1) * f + pad]
                assert blk.min() == blk.max()
                exp[cy, cx] = mask[cy, cx] & blk[0, 0]
        assert (got == exp).all(), f


def test_mask_by_foreground_end_to_end_maskfg():
    """segment_slide(maskfg=1) = the unfiltered masks AND the brute-force filter."""
    w = workload(1)
    slide = make_slide(w.slide).numpy()[:512, :512].copy()
    a0 = arch_string(w.arch)
    w.arch["maskfg"] = 1
    a1 = arch_string(w.arch)
    r0 = op.segment_slide(slide, w.weights(), a0, 64, 128, 64, w.scales, w.classes)
    r1 = op.segment_slide(slide, w.weights(), a1, 64, 128, 64, w.scales, w.classes)
    fg40 = np.kron(r0["fg"], np.ones((8, 8), np.uint8))
    exp = r0["mask"][0] & fg40[64:64 + 512, 64:64 + 512]
    assert (r1["mask"][0] == exp).all()
    assert r1["mask"][0].sum() < r0["mask"][0].sum()
    assert r1["area"][0] == int(exp.sum())


def test_shift_identity_closed_form_five_levels():
    """The 5-level trunk (the bench network's depth, base 8 to keep it cheap) meets the
    shift-identity closed form exactly."""
    a, net, _ = shift_identity_net(5, 8)
    arch = nn.parse_arch(arch_string(a))
    x = np.random.default_rng(8).integers(0, 256, (64, 64, 3)).astype(np.uint8)
    F, E = nn.trunk(net, arch, x)
    assert (F[:, :, :3] == shift_identity_F(x, 5)).all()
    assert (F[:, :, 3:] == 0).all()
