"""Oracle for SURVEY N3: 40x merge of the per-task masks, colour overlay, 10x downsample.

TEST INFRASTRUCTURE ONLY (see oracle/frontend.py header). Plain numpy, following SPEC.md's
render_overlay / downsample_overlay readings of PAPER.md §2.3.
"""
from __future__ import annotations

import numpy as np

# S:381 design decision (the paper says only "different colors"): palette per class index
# TUFT, CAP, PT, DT, PTC, VES (= class codes 0..5, DESIGN R13); alpha 0.4.
PALETTE = np.array([(255, 0, 0), (255, 128, 0), (0, 255, 0), (0, 128, 255), (255, 0, 255), (128, 0, 128)],
                   dtype=np.int64)


def merge_40x(masks, factors, H, W):
    """Nearest-neighbour upsample of each task mask (at its level f: ceil(H/f) x ceil(W/f)) to
    the 40x slide grid: pixel (y, x) takes mask[y // f, x // f] ("the 40x merged
    prediction"). Returns one H x W u8 map per task."""
    out = []
    for m, f in zip(masks, factors):
        ys, xs = np.arange(H) // f, np.arange(W) // f
        out.append(np.asarray(m)[np.ix_(ys, xs)].astype(np.uint8))
    return out


def overlay_40x(slide, masks40, classes):
    """class precedence TUFT > CAP > PT > DT > PTC > VES (lower class code wins);
    a predicted pixel becomes round(0.4 colour + 0.6 base) per channel, others unchanged.
    round(x) with x = (2c + 3b) / 5 is never a half, so it is floor(x + 1/2) = (4c + 6b + 5) // 10."""
    base = np.asarray(slide).astype(np.int64)
    H, W, _ = base.shape
    best = np.full((H, W), 99, np.int64)
    for m, c in zip(masks40, classes):
        best = np.where(np.asarray(m).astype(bool), np.minimum(best, c), best)
    out = base.copy()
    hit = best < 99
    col = PALETTE[np.clip(best, 0, len(PALETTE) - 1)]
    blend = (4 * col + 6 * base + 5) // 10
    out[hit] = blend[hit]
    return out.astype(np.uint8)


def downsample_4(img):
    """factor-4 area average per channel, round half up (sum + n/2) // n; at the
    right / bottom edge a partial block averages the pixels it has (output ceil(H/4) x
    ceil(W/4), DESIGN R15)."""
    a = np.asarray(img).astype(np.int64)
    H, W, C = a.shape
    Ho, Wo = (H + 3) // 4, (W + 3) // 4
    out = np.zeros((Ho, Wo, C), np.int64)
    for by in range(Ho):
        for bx in range(Wo):
            blk = a[4 * by:4 * by + 4, 4 * bx:4 * bx + 4]
            n = blk.shape[0] * blk.shape[1]
            out[by, bx] = (blk.reshape(-1, C).sum(0) + n // 2) // n
    return out.astype(np.uint8)


def downsample_4_fast(img):
    """downsample_4 for images whose sides are multiples of 4 (reshape-sum, no loops)."""
    a = np.asarray(img).astype(np.int64)
    H, W, C = a.shape
    assert H % 4 == 0 and W % 4 == 0
    s = a.reshape(H // 4, 4, W // 4, 4, C).sum((1, 3))
    return ((s + 8) // 16).astype(np.uint8)
