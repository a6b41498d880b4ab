"""Pins of the N3 render oracle (oracle/render.py) against SPEC.md's worked examples
(tests/golden-style literals cited inline) and brute force."""
import numpy as np

from oracle import render as rd


def test_spec_blend_example_and_precedence():
    """base (200,200,200), PT colour (0,255,0), alpha 0.4 -> (120, 222, 120);
    S:365: a pixel in both TUFT and PT maps gets the TUFT colour; no maps -> base."""
    base = np.full((2, 3, 3), 200, np.uint8)
    pt = np.zeros((2, 3), np.uint8)
    pt[0, 0] = 1
    tuft = np.zeros((2, 3), np.uint8)
    tuft[0, 0] = tuft[1, 2] = 1
    out = rd.overlay_40x(base, [pt], [2])
    assert out[0, 0].tolist() == [120, 222, 120]
    assert (out[1] == 200).all() and (out[0, 1:] == 200).all()
    out2 = rd.overlay_40x(base, [pt, tuft], [2, 0])
    tuft_px = [round(0.4 * c + 0.6 * 200) for c in (255, 0, 0)]
    assert out2[0, 0].tolist() == tuft_px and out2[1, 2].tolist() == tuft_px
    assert (rd.overlay_40x(base, [np.zeros((2, 3), np.uint8)], [3]) == base).all()


def test_blend_equals_float_rounding_brute_force():
    rng = np.random.default_rng(3)
    base = rng.integers(0, 256, (17, 19, 3)).astype(np.uint8)
    maps = [rng.integers(0, 2, (17, 19)).astype(np.uint8) for _ in range(6)]
    cls = [5, 1, 3, 0, 4, 2]
    out = rd.overlay_40x(base, maps, cls)
    for y in range(17):
        for x in range(19):
            hits = [c for m, c in zip(maps, cls) if m[y, x]]
            if not hits:
                assert (out[y, x] == base[y, x]).all()
                continue
            col = rd.PALETTE[min(hits)]
            exp = [int(np.floor(0.4 * c + 0.6 * int(b) + 0.5)) for c, b in zip(col, base[y, x])]
            assert out[y, x].tolist() == exp


def test_downsample_spec_examples():
    """constant -> constant at quarter size; a 4x4 block of two colours -> the
    block mean (round half up); the fast path equals the general one."""
    c = np.full((16, 12, 3), 77, np.uint8)
    d = rd.downsample_4(c)
    assert d.shape == (4, 3, 3) and (d == 77).all()
    blk = np.zeros((4, 4, 3), np.uint8)
    blk[:, :2] = (10, 20, 30)
    blk[:, 2:] = (11, 20, 255)
    assert rd.downsample_4(blk)[0, 0].tolist() == [11, 20, 143]  # (21*8+8)//16=11, 20, (285*8+8)//16=143
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, (24, 20, 3)).astype(np.uint8)
    assert (rd.downsample_4(a) == rd.downsample_4_fast(a)).all()
    # ragged edge: partial blocks average what they contain
    e = rng.integers(0, 256, (6, 5, 3)).astype(np.uint8)
    de = rd.downsample_4(e)
    assert de.shape == (2, 2, 3)
    assert de[1, 1].tolist() == [(int(e[4:, 4:, k].sum()) + 1) // 2 for k in range(3)]


def test_merge_40x_nearest():
    m = np.array([[1, 0], [0, 1]], np.uint8)
    up = rd.merge_40x([m], [4], 7, 8)[0]
    assert up.shape == (7, 8)
    assert (up[:4, :4] == 1).all() and (up[:4, 4:] == 0).all() and (up[4:, 4:] == 1).all()
