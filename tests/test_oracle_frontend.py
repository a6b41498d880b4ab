"""Pins for the oracle front end (O1-O6) against the paper / SPEC worked examples,
library routines (SciPy) and textbook definitions -- never against itself."""
import random
from fractions import Fraction

import numpy as np
import pytest
import scipy.ndimage as ndi

from conftest import golden
from oracle import frontend as fe

G = golden("spec_examples.json")


def test_pad_colour_golden():
    g = G["pad_colour_corners"]
    s = np.zeros((4, 4, 3), np.uint8)
    (s[0, 0], s[0, 1], s[1, 0], s[1, 1]) = [np.full(3, v, np.uint8) for v in g["corners"]]
    assert (fe.pad_colour(s) == g["expect"]).all()


def test_pad_colour_round_half_up():
    s = np.zeros((2, 2, 3), np.uint8)
    s[0, 0] = 1  # sum 1 -> (1+2)>>2 = 0 ; sum 2 -> 1 (half up)
    assert (fe.pad_colour(s) == 0).all()
    s[0, 1] = 1
    assert (fe.pad_colour(s) == 1).all()


def test_padded_slide_layout():
    rng = np.random.default_rng(0)
    s = rng.integers(0, 256, (37, 53, 3), dtype=np.uint8)
    p = fe.pad_slide(s, 16)
    assert p.shape == (128, 128, 3)
    assert (p[16:53, 16:69] == s).all()
    pc = fe.pad_colour(s)
    assert (p[0, 0] == pc).all() and (p[-1, -1] == pc).all() and (p[60, 5] == pc).all()


def test_level_golden():
    g = G["pyramid_constant"]
    a = np.full((64, 64, 3), g["value"], np.uint8)
    for f in (2, 4, 8):
        assert (fe.level(a, f) == g["expect"]).all()
    g = G["pyramid_checkerboard"]
    n = g["size"]
    cb = ((np.add.outer(np.arange(n), np.arange(n)) % 2) * 255).astype(np.uint8)
    lv = fe.level(np.repeat(cb[:, :, None], 3, axis=2), g["factor"])
    assert (lv == g["expect"]).all()


@pytest.mark.parametrize("f", [2, 4, 8])
def test_level_brute_force(f):
    rng = np.random.default_rng(f)
    a = rng.integers(0, 256, (3 * f, 5 * f, 3), dtype=np.uint8)
    lv = fe.level(a, f)
    for i in range(3):
        for j in range(5):
            for c in range(3):
                tot = 0
                for y in range(i * f, i * f + f):
                    for x in range(j * f, j * f + f):
                        tot += int(a[y, x, c])
                # round half up of tot / f^2
                q = Fraction(tot, f * f)           # exact mean, rounded half up
                assert lv[i, j, c] == int(np.floor(q + Fraction(1, 2)))


def test_luma_closed_forms():
    px = np.array([[[255, 255, 255], [0, 0, 0], [255, 0, 0], [0, 255, 0], [0, 0, 255],
                    [200, 120, 170]]], np.uint8)
    got = fe.luma(px)[0].tolist()
    # floor((77 R + 150 G + 29 B) / 256)
    assert got == [255, 0, 76, 149, 28, (77 * 200 + 150 * 120 + 29 * 170) // 256]


@pytest.mark.parametrize("k", [3, 5, 7, 9])
def test_median_vs_scipy(k):
    rng = np.random.default_rng(k)
    for trial in range(12):
        h, w = rng.integers(1, 40, 2)
        g = rng.integers(0, 256, (h, w), dtype=np.uint8)
        ref = ndi.median_filter(g, size=k, mode="nearest")
        assert (fe.median_blur(g, k) == ref).all()


def test_median_brute_force_small():
    rng = np.random.default_rng(1)
    g = rng.integers(0, 256, (9, 11), dtype=np.uint8)
    out = fe.median_blur(g, 7)
    for y in range(9):
        for x in range(11):
            vals = sorted(int(g[min(max(y + dy, 0), 8), min(max(x + dx, 0), 10)])
                          for dy in range(-3, 4) for dx in range(-3, 4))
            assert out[y, x] == vals[24]


def test_median_golden():
    g = np.zeros((9, 9), np.uint8)
    g[4, 4] = 255
    assert fe.median_blur(g, G["median_speck"]["aperture"]).max() == G["median_speck"]["expect_max"]
    rng = np.random.default_rng(2)
    a = rng.integers(0, 256, (13, 7), dtype=np.uint8)
    assert (fe.median_blur(a, G["median_identity"]["aperture"]) == a).all()


def _otsu_textbook(hist):
    """Textbook Otsu: t maximising sigma_B^2 = w0 w1 (mu0 - mu1)^2 with exact rationals,
    w_k = class probability, mu_k = class mean; smallest t on ties."""
    N = sum(hist)
    best, bt = None, None
    for t in range(256):
        n0 = sum(hist[: t + 1])
        n1 = N - n0
        if n0 == 0 or n1 == 0:
            continue
        mu0 = Fraction(sum(i * hist[i] for i in range(t + 1)), n0)
        mu1 = Fraction(sum(i * hist[i] for i in range(t + 1, 256)), n1)
        sb = Fraction(n0, N) * Fraction(n1, N) * (mu0 - mu1) ** 2
        if best is None or sb > best:
            best, bt = sb, t
    return bt


def test_otsu_vs_textbook_random():
    rng = random.Random(7)
    for trial in range(1000):
        kind = trial % 4
        h = [0] * 256
        if kind == 0:
            for _ in range(rng.randint(1, 50)):
                h[rng.randrange(256)] += rng.randint(1, 1000)
        elif kind == 1:   # symmetric two-point masses -> ties
            a = rng.randrange(128)
            h[a] = h[255 - a] = rng.randint(1, 9)
            if rng.random() < 0.5:
                h[rng.randrange(256)] += 1
        elif kind == 2:   # dense
            h = [rng.randint(0, 5) for _ in range(256)]
            h[rng.randrange(256)] += 1
        else:             # huge counts (exercise >64-bit products)
            for _ in range(rng.randint(2, 6)):
                h[rng.randrange(256)] += rng.randint(1, 3 * 10 ** 7)
        tb = _otsu_textbook(h)
        if tb is None:
            continue
        assert fe.otsu_threshold(h) == tb, (trial, h)


def test_otsu_golden_and_invariance():
    g = G["otsu_degenerate"]
    h = [0] * 256
    h[g["value"]] = 123
    assert fe.otsu_threshold(h) == g["expect"]
    g = G["otsu_two_mass"]
    h = [0] * 256
    h[g["a"]] = 10
    h[g["b"]] = 30
    t = fe.otsu_threshold(h)
    assert g["lo"] <= t <= g["hi"]
    rng = np.random.default_rng(3)
    for _ in range(50):
        h = rng.integers(0, 100, 256).tolist()
        assert fe.otsu_threshold(h) == fe.otsu_threshold([7 * v for v in h])  # scale invariance


@pytest.mark.parametrize("key", ["plan_tiles_57", "plan_tiles_15"])
def test_origins_golden(key):
    g = G[key]
    assert len(fe.origins(g["E"], g["P"], g["S"])) == g["expect"]


def test_origins_closed_form_random():
    rng = np.random.default_rng(4)
    for _ in range(500):
        P = int(rng.integers(1, 600))
        S = int(rng.integers(1, P + 1))
        E = int(rng.integers(P, 5000))
        o = fe.origins(E, P, S)
        # closed form: ceil((E-P)/S) + 1 origins, last one E-P, all < E-P+1, strictly increasing
        assert len(o) == -(-(E - P) // S) + 1
        assert o[0] == 0 and o[-1] == E - P and all(b > a for a, b in zip(o, o[1:]))
        assert all(b - a <= S for a, b in zip(o, o[1:]))


def test_grid_sizes_golden():
    gr = golden("grids.json")
    for key, g in gr.items():
        if key.startswith("_"):
            continue
        Hp, Wp = fe.padded_extent(g["H"], g["W"], g["pad"])
        if "grids" in g:
            for f, (ny, nx) in g["grids"].items():
                f = int(f)
                assert len(fe.origins(Hp // f, g["P"], g["S"])) == ny
                assert len(fe.origins(Wp // f, g["P"], g["S"])) == nx
        for f, tot in g.get("totals", {}).items():
            f = int(f)
            n = len(fe.origins(Hp // f, g["P"], g["S"])) * len(fe.origins(Wp // f, g["P"], g["S"]))
            assert n == tot, (key, f)


def test_tile_plan_vs_summed_area_table():
    """Keep test recomputed with an independent summed-area table."""
    rng = np.random.default_rng(5)
    Hp, Wp, P, S = 1024, 1280, 128, 64
    fg = (rng.random((Hp // 8, Wp // 8)) < 0.004).astype(np.uint8)
    fg[40:60, 30:90] = 1
    sat = np.zeros((fg.shape[0] + 1, fg.shape[1] + 1), np.int64)
    sat[1:, 1:] = fg.cumsum(0).cumsum(1)
    kept, grids = fe.tile_plan(fg, Hp, Wp, [1, 2, 4, 8], P, S)
    exp = []
    for f in (8, 4, 2, 1):
        for oy in fe.origins(Hp // f, P, S):
            for ox in fe.origins(Wp // f, P, S):
                y0, x0, n = oy * f // 8, ox * f // 8, P * f // 8
                c = sat[y0 + n, x0 + n] - sat[y0, x0 + n] - sat[y0 + n, x0] + sat[y0, x0]
                if c * 100 >= n * n:
                    exp.append((f, oy, ox))
    assert kept == exp
    assert len(kept) > 0


def test_blank_slide_no_tiles():
    """north_star invariant: all-background slides yield empty masks (no kept tiles)."""
    from omniseg_inputs import blank_slide
    s = blank_slide(1024, 1024).numpy()
    p = fe.pad_slide(s, 128)
    det = fe.detection(p, 1024, 1024, 128)
    assert det["fg"].sum() == 0
    kept, _ = fe.tile_plan(det["fg"], p.shape[0], p.shape[1], [1], 256, 128)
    assert kept == []


def test_all_tissue_full_grid():
    """Uniform tissue tone 120 (top-left 2x2 light, so the pad colour is light and the
    guard 240-16 passes tone 120). The 7x7 median with edge replication only turns the
    interior's corner pixels (>= 25 of 49 window pixels in the pad) light, so Otsu
    splits the tissue tone from those, every other interior pixel is foreground, and
    every tile whose footprint overlaps the interior is kept: the full 5x5 grid
    (per-axis overlaps 8,16,16,16,8 level-8 px of a 16 px footprint)."""
    s = np.full((512, 512, 3), 120, np.uint8)
    s[:2, :2] = 240
    p = fe.pad_slide(s, 64)
    det = fe.detection(p, 512, 512, 64)
    assert 120 <= det["t"] < 240
    assert det["fg"].sum() >= 64 * 64 - 4 * 9 and det["fg"][:8].sum() == 0
    kept, grids = fe.tile_plan(det["fg"], p.shape[0], p.shape[1], [1], 128, 128)
    assert grids[1] == (5, 5, 25) and len(kept) == 25


def test_chunked_detection_equals_whole_frame():
    """The memory-bounded evaluation (row windows) equals the whole-frame definition."""
    from omniseg_inputs import make_slide, workload
    w = workload(1)
    s = make_slide(w.slide).numpy()
    p = fe.pad_slide(s, w.pad)
    a = fe.detection(p, 1024, 1024, w.pad)
    b = fe.detection_chunked(s, w.pad, rows_per_chunk=256)
    assert a["t"] == b["t"] and (a["fg"] == b["fg"]).all() and (a["hist"] == b["hist"]).all()
    assert a["g_pad"] == b["g_pad"]
    L1 = fe.level(p, 4)
    assert (fe.level_window(s, w.pad, fe.pad_colour(s), 4, 40, 12, 64) == L1[40:104, 12:76]).all()


# ---------------------------------------------------------------- tiny-component removal
def _flood_components(mask):
    """Brute-force 4-connected components (explicit BFS), independent of scipy."""
    H, W = mask.shape
    lab = -np.ones((H, W), np.int64)
    sizes = []
    for y in range(H):
        for x in range(W):
            if mask[y, x] and lab[y, x] < 0:
                k = len(sizes)
                stack, n = [(y, x)], 0
                lab[y, x] = k
                while stack:
                    cy, cx = stack.pop()
                    n += 1
                    for ny, nx in ((cy - 1, cx), (cy + 1, cx), (cy, cx - 1), (cy, cx + 1)):
                        if 0 <= ny < H and 0 <= nx < W and mask[ny, nx] and lab[ny, nx] < 0:
                            lab[ny, nx] = k
                            stack.append((ny, nx))
                sizes.append(n)
    return lab, sizes


def test_drop_small_components_matches_flood_fill():
    rng = np.random.default_rng(11)
    for trial in range(20):
        m = (rng.random((23, 31)) < 0.45).astype(np.uint8)
        lab, sizes = _flood_components(m)
        for min_area in (1, 2, 3, 5, 9):
            ref = np.zeros_like(m)
            for k, n in enumerate(sizes):
                if n >= min_area:
                    ref[lab == k] = 1
            assert (fe.drop_small_components(m, min_area) == ref).all(), (trial, min_area)


def test_drop_small_components_spec_example_and_invariants():
    """one large dark disk + a 3-pixel speck, min area above 3 -> exactly the disk
    survives; diagonal-only contact does not connect (4-connectivity); filtering only removes;
    blank stays blank."""
    m = np.zeros((64, 64), np.uint8)
    yy, xx = np.mgrid[:64, :64]
    m[(yy - 30) ** 2 + (xx - 30) ** 2 <= 15 ** 2] = 1
    m[2, 60:63] = 1                                   # 3-pixel speck
    m[50, 50] = m[51, 51] = 1                         # diagonal pair = two 1-px components
    out = fe.drop_small_components(m, 4)
    assert out[2, 60:63].sum() == 0 and out[50, 50] == 0 and out[51, 51] == 0
    assert (out[(yy - 30) ** 2 + (xx - 30) ** 2 <= 15 ** 2] == 1).all()
    assert (out <= m).all()
    assert fe.drop_small_components(np.zeros((8, 8), np.uint8), 5).sum() == 0
    assert (fe.drop_small_components(m, 0) == m).all()
