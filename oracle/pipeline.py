"""Oracle, end to end: segment_slide (O1-O11) and sampled-pixel evaluation.

TEST INFRASTRUCTURE ONLY (see oracle/frontend.py header).
"""
from __future__ import annotations

import numpy as np

from . import frontend as fe
from . import net as nn


def task_factors(arch: dict, scales):
    """Per task: level factor f = slide_mag / scale (§1: 40x/10x/5x copies
    of the 40x scan; f in {1,2,4,8}) and the scale index."""
    out = []
    for s in scales:
        if s not in arch["scale_codes"] or arch["slide_mag"] % s:
            raise ValueError(f"scale {s} not in scale_codes")
        f = arch["slide_mag"] // s
        if f not in (1, 2, 4, 8):
            raise ValueError("level factor must be 1, 2, 4 or 8")
        out.append((f, arch["scale_codes"].index(s)))
    return out


def front_end(slide: np.ndarray, pad: int, patch: int, stride: int, factors, min_area: int = 0):
    """O1-O6: pad colour, padded frame, level-8 detection (+ the optional tiny-component
    removal), tile plan."""
    H, W, _ = slide.shape
    padded = fe.pad_slide(slide, pad)
    Hp, Wp = padded.shape[:2]
    det = fe.detection(padded, H, W, pad, min_area=min_area)
    kept, grids = fe.tile_plan(det["fg"], Hp, Wp, factors, patch, stride)
    return dict(padded=padded, Hp=Hp, Wp=Wp, det=det, kept=kept, grids=grids,
                pc=fe.pad_colour(slide))


def canvas_shape(H, W, f):
    """Task canvas at the task's own scale over the unpadded slide: ceil(H/f) x ceil(W/f)
    (§2.3 'merged back into an image the original size'; at task scale, DESIGN R10)."""
    return (H + f - 1) // f, (W + f - 1) // f


def segment_slide(slide: np.ndarray, blob, arch_s: str, pad: int, patch: int, stride: int,
                  scales, classes, progress=None, fusion=None, keep_windows=False):
    """Plain CPU pipeline. Returns dict with per-task prob (float64),
    mask (u8), area (int), the kept tile list, fg mask and Otsu t.
    fusion: "mean" (overlap-weighted mean of p, DESIGN R11) or "vote" (hard majority vote,
    SURVEY N1: each window votes p >= 1/2, "majority of the testing results", "1 of
    2" / "4 of 8" -- both "at least half"); default: the arch string's `fusion` key, else mean.
    With the arch key vthr (one vote count per scale code) the vote mask is the paper's literal
    count threshold instead (finalize_vote_count). keep_windows: also return every kept window's
    per-task probability maps, {(f, oy, ox): {task index: p}} (for tests that inspect votes)."""
    arch = nn.parse_arch(arch_s)
    if fusion is None:
        fusion = arch.get("fusion", "mean")
    if fusion not in ("mean", "vote"):
        raise ValueError("fusion must be mean or vote")
    net = nn.unpack_weights(arch, blob)
    H, W, _ = slide.shape
    tf = task_factors(arch, scales)
    fr = front_end(slide, pad, patch, stride, [f for f, _ in tf], min_area=arch.get("fgmin", 0))
    levels = {f: fe.level(fr["padded"], f) for f in set(f for f, _ in tf)}
    sums, cnts, windows = [], [], {}
    for (f, _s) in tf:
        sums.append(np.zeros(canvas_shape(H, W, f)))
        cnts.append(np.zeros(canvas_shape(H, W, f), np.int64))
    for i, (f, oy, ox) in enumerate(fr["kept"]):
        tile = levels[f][oy:oy + patch, ox:ox + patch]
        tasks = [(t, classes[t], s) for t, (ft, s) in enumerate(tf) if ft == f]
        p = nn.predict_tile(net, arch, tile, [(c, s) for _, c, s in tasks])
        if keep_windows:
            windows[(f, oy, ox)] = {t: p[k] for k, (t, _c, _s) in enumerate(tasks)}
        for k, (t, _c, _s) in enumerate(tasks):
            val = vote_of(p[k]) if fusion == "vote" else p[k]
            stitch_add(sums[t], cnts[t], val, oy - pad // f, ox - pad // f)
        if progress:
            progress(i, len(fr["kept"]))
    vthr = arch.get("vthr")
    if vthr is not None and len(vthr) != len(arch["scale_codes"]):
        raise ValueError("vthr needs one threshold per scale code")
    probs, masks, areas = [], [], []
    for t in range(len(tf)):
        thr = vthr[tf[t][1]] if (fusion == "vote" and vthr) else 0
        if thr > 0:
            prob, mask = finalize_vote_count(sums[t], cnts[t], thr)
        else:
            prob, mask = finalize(sums[t], cnts[t])
        if arch.get("maskfg", 0):
            mask = mask_by_foreground(mask, fr["det"]["fg"], tf[t][0], pad)
        probs.append(prob)
        masks.append(mask)
        areas.append(int(mask.sum()))
    return dict(prob=probs, mask=masks, area=areas, kept=fr["kept"], grids=fr["grids"],
                fg=fr["det"]["fg"], t=fr["det"]["t"], hist=fr["det"]["hist"],
                g_pad=fr["det"]["g_pad"], cnt=cnts, windows=windows if keep_windows else None)


def vote_of(p):
    """A window's binary vote per pixel: p >= 1/2 (P:97 thresholds)."""
    return (np.asarray(p) >= 0.5).astype(np.float64)


def stitch_add(acc_sum, acc_cnt, p, y0, x0):
    """Overlap-weighted accumulation (P:69 overlap tiling, P:87 merge; north_star
    'stitched back into a slide-level canvas by overlap-weighted accumulation'):
    add p and a unit weight to every canvas pixel the tile covers; (y0, x0) is the
    tile origin in canvas coordinates (may be negative / run past the edge)."""
    Hc, Wc = acc_sum.shape
    P = p.shape[0]
    ys, ye = max(0, y0), min(Hc, y0 + P)
    xs, xe = max(0, x0), min(Wc, x0 + P)
    if ys >= ye or xs >= xe:
        return
    acc_sum[ys:ye, xs:xe] += p[ys - y0:ye - y0, xs - x0:xe - x0]
    acc_cnt[ys:ye, xs:xe] += 1


def finalize(acc_sum, acc_cnt):
    """prob = sum / cnt (0 where no kept tile covers the pixel); mask = prob >= 0.5
    (the paper's 1-of-2 and 4-of-8 votes are both 'at least half'; DESIGN R11)."""
    prob = np.where(acc_cnt > 0, acc_sum / np.maximum(acc_cnt, 1), 0.0)
    return prob, (prob >= 0.5).astype(np.uint8)


def finalize_vote_count(votes, cnt, thr):
    """Hard vote with the paper's literal vote-count threshold (arch key vthr; "the major
    vote threshold was set to 1" at 40x, "set to 4" at 10x / 5x; S:266-268, S:310-311 read
    against the 2-D coverage): mask = votes >= min(thr, coverage), coverage > 0 (min() keeps
    edge pixels covered by fewer windows than thr decidable). prob = vote fraction."""
    prob = np.where(cnt > 0, votes / np.maximum(cnt, 1), 0.0)
    mask = (cnt > 0) & (votes >= np.minimum(thr, cnt))
    return prob, mask.astype(np.uint8)


def mask_by_foreground(mask, fg8, f, pad):
    """P:87 §2.3 "the foreground contour generated during tissue detection was utilized again to
    filter out noises from the prediction"; S:350 filter_by_foreground: map AND mask with the
    mask nearest-neighbour rescaled. Canvas pixel (cy, cx) of a task at level f
    is padded-40x pixel (cy f + pad, cx f + pad), i.e. level-8 pixel ((cy f + pad) // 8, ...)."""
    Ht, Wt = mask.shape
    ys = (np.arange(Ht) * f + pad) // 8
    xs = (np.arange(Wt) * f + pad) // 8
    return (mask.astype(bool) & fg8[np.ix_(ys, xs)].astype(bool)).astype(np.uint8)


def covering_tiles(kept, f, pad, patch, cy, cx):
    """Kept tiles of scale f whose window covers canvas pixel (cy, cx) of a task at f."""
    py, px = cy + pad // f, cx + pad // f
    return [(ff, oy, ox) for (ff, oy, ox) in kept
            if ff == f and oy <= py < oy + patch and ox <= px < ox + patch]
