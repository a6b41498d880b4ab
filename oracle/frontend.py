"""Oracle, front end: padding, pyramid, tissue detection, tile plan (O1-O6).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product
path (paper_2305_14566_b200) never imports, calls or links it.

Plain, slow, obviously correct numpy; every step is integer-exact. Each
function cites the passage it follows: P:L = /root/reference/PAPER.md line L
(plus its section), S:L = SPEC.md line L, SURVEY Ox = SURVEY.md §8(c) row Ox.
Where the paper is silent the reading is the one DESIGN.md §2 lists.
"""
from __future__ import annotations

import numpy as np


def pad_colour(slide: np.ndarray) -> np.ndarray:
    """P:59 §2.1 / P:96 §3.2 "mean of a 2x2 image vector on the top-left corner";
    per channel, rounded half up: (s00+s01+s10+s11+2)>>2.  [SURVEY O1]"""
    blk = slide[:2, :2, :].astype(np.int64)
    return (blk.sum(axis=(0, 1)) + 2) // 4


def padded_extent(H: int, W: int, pad: int):
    """Padded frame (§2.1, padding added on every side). Bottom/right
    are further rounded up to a multiple of 128 px (reading R2). [SURVEY O2]"""
    r = lambda v: (v + 127) // 128 * 128  # noqa: E731
    return r(H + 2 * pad), r(W + 2 * pad)


def pad_slide(slide: np.ndarray, pad: int) -> np.ndarray:
    """Materialise the padded slide: slide at offset (pad, pad), everything else the
    pad colour."""
    H, W, _ = slide.shape
    Hp, Wp = padded_extent(H, W, pad)
    out = np.empty((Hp, Wp, 3), np.uint8)
    out[:, :] = pad_colour(slide).astype(np.uint8)
    out[pad:pad + H, pad:pad + W] = slide
    return out


def level(padded: np.ndarray, f: int) -> np.ndarray:
    """Area-mean downsample by f, computed directly from 40x (not cascaded), per
    channel, rounded half up: (sum + f^2/2) // f^2.  P:67 §2.2 / P:92 §3.1 (40x, 10x,
    5x copies of the 40x scan); interpolation unstated in the paper -> area mean
    (S:46). [SURVEY O3]"""
    if f == 1:
        return padded.copy()
    Hp, Wp, C = padded.shape
    assert Hp % f == 0 and Wp % f == 0
    s = padded.astype(np.int64).reshape(Hp // f, f, Wp // f, f, C).sum(axis=(1, 3))
    return ((s + (f * f) // 2) // (f * f)).astype(np.uint8)


def luma(rgb: np.ndarray) -> np.ndarray:
    """Integer luma (77R + 150G + 29B) >> 8 (weights 77/150/29 over 256)."""
    v = rgb.astype(np.int64)
    return ((77 * v[..., 0] + 150 * v[..., 1] + 29 * v[..., 2]) >> 8).astype(np.uint8)


def median_blur(g: np.ndarray, k: int) -> np.ndarray:
    """k x k median with edge replication (§3.2 "Median blur ... threshold set to
    59", read as the aperture, scaled to the detection level: k=7 at 5x).
    The median of k*k (odd) integers is the element of rank (k*k)//2."""
    assert k % 2 == 1 and k >= 1
    r = k // 2
    p = np.pad(g, r, mode="edge")
    win = np.lib.stride_tricks.sliding_window_view(p, (k, k))
    flat = win.reshape(g.shape[0], g.shape[1], k * k)
    return np.partition(flat, (k * k) // 2, axis=-1)[..., (k * k) // 2].astype(np.uint8)


def otsu_threshold(hist) -> int:
    """Otsu threshold (§2.1, "Ostu edge detection"), S:115-119:
    smallest t maximising the between-class variance of {<=t} vs {>t}.

    With n0 = sum_{i<=t} h_i, m0 = sum_{i<=t} i h_i, N = sum h, M = sum i h:
    sigma_B^2(t) = (N m0 - M n0)^2 / (N^2 n0 (N - n0)); the constant N^2 is dropped.
    Exact with Python integers (cross-multiplied compare). Candidates need
    0 < n0 < N; with none (a single-valued histogram) the answer is that value
    (S:119). An empty histogram returns 255 (nothing is darker-than-or-equal and
    tissue needs pixels anyway)."""
    h = [int(v) for v in hist]
    N = sum(h)
    M = sum(i * v for i, v in enumerate(h))
    if N == 0:
        return 255
    best_t, best_num, best_den = None, 0, 1
    n0 = m0 = 0
    for t in range(256):
        n0 += h[t]
        m0 += t * h[t]
        if n0 == 0 or n0 == N:
            continue
        num = (N * m0 - M * n0) ** 2
        den = n0 * (N - n0)
        if best_t is None or num * best_den > best_num * den:
            best_t, best_num, best_den = t, num, den
    if best_t is None:
        return next(i for i, v in enumerate(h) if v)
    return best_t


def detection(padded: np.ndarray, H: int, W: int, pad: int, k: int = 7, guard: int = 16, min_area: int = 0):
    """Tissue detection at 5x = level 8. [SURVEY O4-O5]

    Returns dict(g8 = luma of level 8, gm = median-blurred luma, hist (interior),
    t = Otsu threshold, g_pad = luma of the pad colour, fg = foreground mask u8).
    Interior = level-8 rows [pad/8, pad/8 + H//8), cols likewise (pixels wholly
    inside the slide). fg = interior & gm <= t & gm <= g_pad - guard (tissue is the
    darker side; the guard is DESIGN.md reading R7)."""
    assert pad % 8 == 0
    L8 = level(padded, 8)
    g8 = luma(L8)
    gm = median_blur(g8, k)
    r0, c0 = pad // 8, pad // 8
    r1, c1 = r0 + H // 8, c0 + W // 8
    interior = np.zeros(gm.shape, bool)
    interior[r0:r1, c0:c1] = True
    hist = np.bincount(gm[interior].ravel(), minlength=256).astype(np.int64)
    t = otsu_threshold(hist)
    pc = padded[0, 0]
    g_pad = int(luma(pc[None, None, :])[0, 0])
    fg = interior & (gm.astype(np.int64) <= t) & (gm.astype(np.int64) <= g_pad - guard)
    if min_area > 0:  # SURVEY N2 (arch fgmin): components below min_area level-8 pixels dropped
        fg = drop_small_components(fg, min_area)
    return dict(g8=g8, gm=gm, hist=hist, t=t, g_pad=g_pad, fg=fg.astype(np.uint8))


def drop_small_components(fg: np.ndarray, min_area: int) -> np.ndarray:
    """Tiny-noise removal ("the foreground contour was set to a certain threshold to
    remove tiny noises"; S:124-127 detect_foreground: 4-connected components, drop those
    below min_component_area). Labelling by scipy.ndimage.label with the
    4-neighbour cross (a library primitive, pinned against a brute-force flood fill in
    tests/test_oracle_frontend.py); keep components with >= min_area pixels."""
    from scipy import ndimage
    fg = np.asarray(fg).astype(bool)
    if min_area <= 0 or not fg.any():
        return fg.astype(np.uint8)
    lab, _ = ndimage.label(fg, structure=[[0, 1, 0], [1, 1, 1], [0, 1, 0]])
    sizes = np.bincount(lab.ravel())
    keep = sizes >= min_area
    keep[0] = False
    return keep[lab].astype(np.uint8)


def origins(E: int, P: int, S: int):
    """Tile origins along one axis of extent E: 0, S, 2S, ... <= E-P, plus a clamped
    final origin E-P if not already present (P:69 overlap tiling)."""
    if P > E:
        raise ValueError("window larger than extent")
    o = list(range(0, E - P + 1, S))
    if o[-1] != E - P:
        o.append(E - P)
    return o


def tile_plan(fg: np.ndarray, Hp: int, Wp: int, factors, P: int, S: int):
    """Candidate grids per scale and the keep test ("remove blank regions";
    S:133-141 region_is_tissue with min_fraction 0.01 = S:151, out-of-bounds =
    background). A tile at level f with origin (oy, ox) covers level-8 rows
    [oy f/8, (oy+P) f/8) (cols likewise); kept iff 100 * (#fg in it) >= (P f / 8)^2.

    Order: scale descending (coarsest first), then row, then column.
    Returns list of (f, oy, ox) kept, and per-f (ny, nx, kept_count)."""
    kept, grids = [], {}
    for f in sorted(set(factors), reverse=True):
        Ey, Ex = Hp // f, Wp // f
        oys, oxs = origins(Ey, P, S), origins(Ex, P, S)
        area = (P * f // 8) ** 2
        n = 0
        for oy in oys:
            for ox in oxs:
                assert (oy * f) % 8 == 0 and (ox * f) % 8 == 0
                y0, x0 = oy * f // 8, ox * f // 8
                cnt = int(fg[y0:y0 + P * f // 8, x0:x0 + P * f // 8].sum())
                if 100 * cnt >= area:
                    kept.append((f, oy, ox))
                    n += 1
        grids[f] = (len(oys), len(oxs), n)
    return kept, grids


def padded_window(slide: np.ndarray, pad: int, pc, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    """Rows [r0, r1) x cols [c0, c1) of the padded slide (pad_slide) without materialising
    the whole frame: slide pixels where they exist, the pad colour elsewhere."""
    H, W, _ = slide.shape
    out = np.empty((r1 - r0, c1 - c0, 3), np.uint8)
    out[:, :] = np.asarray(pc, np.uint8)
    ys, ye = max(r0, pad), min(r1, pad + H)
    xs, xe = max(c0, pad), min(c1, pad + W)
    if ys < ye and xs < xe:
        out[ys - r0:ye - r0, xs - c0:xe - c0] = slide[ys - pad:ye - pad, xs - pad:xe - pad]
    return out


def detection_chunked(slide: np.ndarray, pad: int, rows_per_chunk: int = 4096, k: int = 7, guard: int = 16):
    """`detection` evaluated on a padded frame too large to materialise: level 8 is a
    block-local mean, so computing it over row windows that are multiples of 8 rows and
    concatenating is identical to `level(pad_slide(slide), 8)`; the median, histogram,
    Otsu and foreground then run on the (small) whole level-8 grid exactly as in
    `detection`."""
    H, W, _ = slide.shape
    Hp, Wp = padded_extent(H, W, pad)
    pc = pad_colour(slide)
    step = rows_per_chunk // 8 * 8
    L8 = np.concatenate([level(padded_window(slide, pad, pc, r, min(Hp, r + step), 0, Wp), 8)
                         for r in range(0, Hp, step)])
    g8 = luma(L8)
    gm = median_blur(g8, k)
    r0, c0 = pad // 8, pad // 8
    r1, c1 = r0 + H // 8, c0 + W // 8
    interior = np.zeros(gm.shape, bool)
    interior[r0:r1, c0:c1] = True
    hist = np.bincount(gm[interior].ravel(), minlength=256).astype(np.int64)
    t = otsu_threshold(hist)
    g_pad = int(luma(pc.astype(np.uint8)[None, None, :])[0, 0])
    fg = interior & (gm.astype(np.int64) <= t) & (gm.astype(np.int64) <= g_pad - guard)
    return dict(g8=g8, gm=gm, hist=hist, t=t, g_pad=g_pad, fg=fg.astype(np.uint8), pc=pc, Hp=Hp, Wp=Wp)


def level_window(slide: np.ndarray, pad: int, pc, f: int, oy: int, ox: int, P: int) -> np.ndarray:
    """The P x P window at level f with origin (oy, ox) (level-f padded coordinates),
    computed from the 40x padded region it averages (identical to slicing `level`)."""
    win = padded_window(slide, pad, pc, oy * f, (oy + P) * f, ox * f, (ox + P) * f)
    return level(win, f)
