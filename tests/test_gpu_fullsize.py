"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times
(fp16f8, batch 64, device-resident slide and outputs):

* front end bit-exact at full size: Otsu t, g_pad, the level-8 foreground mask and the
  kept-tile list, against the oracle's detection (evaluated row-chunked, identical to the
  whole-frame definition: tests/test_oracle_frontend.py) and tile plan;
* the probability canvas on sampled pixels that the oracle computes one by one (every
  kept window covering the pixel through the fp64 trunk + head, averaged): |dp| <= 1e-2,
  and the mask agrees wherever the oracle probability is not within 1e-2 of 1/2.
"""
import numpy as np
import pytest
import torch

from omniseg_inputs import arch_string, geometry, render, workload
from oracle import frontend as fe
from oracle import net as nn
from oracle import pipeline as op

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _unpack(ids, Hp, Wp, P, S):
    out = []
    for v in ids.tolist():
        f = 1 << (v >> 30)
        out.append((f, min(((v >> 15) & 0x7FFF) * S, Hp // f - P), min((v & 0x7FFF) * S, Wp // f - P)))
    return out


def _region_check(kept, f, pad, P, S, Ht, Wt, rng, pt_tasks, masks, want):
    """Pick up to `want` kept windows K of scale f; each K's sub-square [S/2, S) x [S/2, S)
    (window-relative) lies in K and the windows one stride up / left only (S = P/2), so a
    handful of windows covers every pixel of it. Yields (region slices, covering windows)."""
    ks = [k for k in kept if k[0] == f]
    order = rng.permutation(len(ks))
    # prefer windows whose region holds positive mask pixels of the first task (informative)
    def region(k):
        y0, x0 = k[1] - pad // f + S // 2, k[2] - pad // f + S // 2
        return max(0, y0), min(Ht, y0 + S // 2), max(0, x0), min(Wt, x0 + S // 2)
    scored = []
    for i in order[:400]:
        y0, y1, x0, x1 = region(ks[i])
        if y1 - y0 < 16 or x1 - x0 < 16:
            continue
        scored.append((-int(masks[0][y0:y1, x0:x1].sum() > 0), int(i)))
    scored.sort()
    out = []
    for _, i in scored:
        y0, y1, x0, x1 = region(ks[i])
        py0, py1, px0, px1 = y0 + pad // f, y1 + pad // f, x0 + pad // f, x1 + pad // f
        cov = [k for k in ks if k[1] < py1 and k[1] + P > py0 and k[2] < px1 and k[2] + P > px0]
        if len(cov) > 6:
            continue
        out.append(((y0, y1, x0, x1), cov))
        if len(out) == want:
            break
    return out


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fullsize_front_end_and_sampled_probabilities(gpu_lib, cfg):
    """Full-size bit-exact front end, then, for EVERY task (every scale: 5x f = 8, 10x f = 4,
    40x f = 1 on cfg3/cfg4), element-wise probability/mask checks over whole sub-squares of
    kept windows whose covering windows the fp64 oracle computes (two regions per scale,
    <= 6 oracle windows each): |dp| <= 1e-2, masks equal except where the oracle p is within
    1e-2 of 1/2; >= 500 checked pixels per task (printed)."""
    from paper_2305_14566_b200 import Omniseg
    w = workload(cfg)
    H, W, P, S, pad = w.H, w.W, w.patch, w.stride, w.pad
    slide_d = render(geometry(w.slide), device="cuda", chunk_rows=2048)
    slide = slide_d.cpu().numpy()
    h = Omniseg(arch_string(w.arch), w.weights())
    sizes = [h.output_size(H, W, s) for s in w.scales]
    prob = torch.empty(sum(sizes), dtype=torch.float32, device="cuda")
    mask = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
    h.segment_slide(slide_d, H, W, pad, P, S, w.scales, w.classes, prob, mask, None)
    torch.cuda.synchronize()
    prob, mask = prob.cpu().numpy(), mask.cpu().numpy()
    # ---- front end, bit-exact
    det = fe.detection_chunked(slide, pad)
    fg, t, gpad = h.fgmask()
    assert t == det["t"] and gpad == det["g_pad"]
    assert (fg == det["fg"]).all()
    arch = nn.parse_arch(arch_string(w.arch))
    tf = op.task_factors(arch, w.scales)
    kept, _ = fe.tile_plan(det["fg"], det["Hp"], det["Wp"], [f for f, _ in tf], P, S)
    got = _unpack(h.tiles(), det["Hp"], det["Wp"], P, S)
    assert got == kept
    # ---- element-wise regions, per scale (tasks of one scale share the windows)
    net = nn.unpack_weights(arch, w.weights())
    rng = np.random.default_rng(cfg)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    checked = [0] * len(tf)
    worst = [0.0] * len(tf)
    for f in sorted(set(f for f, _ in tf), reverse=True):
        tids = [ti for ti, (ft, _) in enumerate(tf) if ft == f]
        Ht, Wt = (H + f - 1) // f, (W + f - 1) // f
        pts = [prob[offs[ti]:offs[ti + 1]].reshape(Ht, Wt) for ti in tids]
        mts = [mask[offs[ti]:offs[ti + 1]].reshape(Ht, Wt) for ti in tids]
        cache = {}
        for (y0, y1, x0, x1), cov in _region_check(kept, f, pad, P, S, Ht, Wt, rng, pts, mts, 2):
            for k in cov:
                if k not in cache:
                    win = fe.level_window(slide, pad, det["pc"], f, k[1], k[2], P)
                    Fr, Er = nn.trunk(net, arch, win)
                    g = nn.gap(Er)
                    cache[k] = {ti: nn.head(Fr, nn.controller(net, arch, g, w.classes[ti], tf[ti][1])) for ti in tids}
            for j, ti in enumerate(tids):
                acc = np.zeros((y1 - y0, x1 - x0))
                cnt = np.zeros((y1 - y0, x1 - x0), np.int64)
                for k in cov:
                    oy, ox = k[1] - pad // f, k[2] - pad // f   # window origin in canvas coordinates
                    a0, a1 = max(y0, oy), min(y1, oy + P)
                    b0, b1 = max(x0, ox), min(x1, ox + P)
                    acc[a0 - y0:a1 - y0, b0 - x0:b1 - x0] += cache[k][ti][a0 - oy:a1 - oy, b0 - ox:b1 - ox]
                    cnt[a0 - y0:a1 - y0, b0 - x0:b1 - x0] += 1
                assert (cnt > 0).all()
                p_ref = acc / cnt
                p_gpu = pts[j][y0:y1, x0:x1].astype(np.float64)
                m_gpu = mts[j][y0:y1, x0:x1]
                d = np.abs(p_gpu - p_ref)
                assert d.max() <= 1e-2, (cfg, ti, f, d.max())
                dis = m_gpu != (p_ref >= 0.5)
                assert (np.abs(p_ref[dis] - 0.5) <= 1e-2).all(), (cfg, ti, "mask flip away from 1/2")
                checked[ti] += d.size
                worst[ti] = max(worst[ti], float(d.max()))
    print(f"cfg{cfg}: checked px per task {checked}, max |dp| per task {[f'{v:.2e}' for v in worst]}")
    assert min(checked) >= 500, checked


def test_synthetic_slide_cpu_gpu_identical(gpu_lib):
    """The seeded generator gives byte-identical windows on CPU and GPU (bench generates
    slides on the GPU, the oracle side on the CPU)."""
    for cfg in (3, 4, 5):
        g = geometry(workload(cfg).slide)
        for (r0, c0) in ((0, 0), (5000, 3000), (g["H"] - 300, g["W"] - 700)):
            a = render(g, r0, r0 + 256, c0, c0 + 512).numpy()
            b = render(g, r0, r0 + 256, c0, c0 + 512, device="cuda").cpu().numpy()
            assert (a == b).all(), (cfg, r0, c0)


def test_fullsize_paper_geometry_vote_sampled(gpu_lib):
    """SURVEY N1 at full size, in bench.py's `cfg4_paper` launch configuration (cfg4 slide,
    vote fusion, 40x windows at S = 256 and 10x / 5x windows at S = 64, one call per stride):
    each call's tile plan bit-exact against the oracle's; on sampled pixels (chosen where few
    kept windows cover them, so the fp64 oracle stays cheap) the vote fraction equals the
    oracle's count of windows with p >= 1/2, except where a window's oracle p is within 1e-2
    of 1/2 (its vote may flip under fp16f8 rounding)."""
    import importlib.util
    import os
    from paper_2305_14566_b200 import Omniseg
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    w, groups = bench.resolve_workload("cfg4_paper")
    H, W, P, pad = w.H, w.W, w.patch, w.pad
    slide_d = render(geometry(w.slide), device="cuda", chunk_rows=2048)
    slide = slide_d.cpu().numpy()
    det = fe.detection_chunked(slide, pad)
    arch = nn.parse_arch(arch_string(w.arch))
    assert arch["fusion"] == "vote"
    net = nn.unpack_weights(arch, w.weights())
    h = Omniseg(arch_string(w.arch), w.weights())
    rng = np.random.default_rng(41)
    checked = 0
    for S, idx in groups:
        scales = [w.scales[i] for i in idx]
        classes = [w.classes[i] for i in idx]
        tf = op.task_factors(arch, scales)
        sizes = [h.output_size(H, W, s) for s in scales]
        prob = torch.empty(sum(sizes), dtype=torch.float32, device="cuda")
        mask = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
        h.segment_slide(slide_d, H, W, pad, P, S, scales, classes, prob, mask, None)
        torch.cuda.synchronize()
        prob, mask = prob.cpu().numpy(), mask.cpu().numpy()
        kept, _ = fe.tile_plan(det["fg"], det["Hp"], det["Wp"], [f for f, _ in tf], P, S)
        assert _unpack(h.tiles(), det["Hp"], det["Wp"], P, S) == kept
        offs = np.concatenate([[0], np.cumsum(sizes)])
        cache = {}
        for ti, (f, s_idx) in enumerate(tf):
            Ht, Wt = (H + f - 1) // f, (W + f - 1) // f
            pt = prob[offs[ti]:offs[ti + 1]].reshape(Ht, Wt)
            mt = mask[offs[ti]:offs[ti + 1]].reshape(Ht, Wt)
            cov = np.argwhere(pt > 0)
            cand = [tuple(cov[i]) for i in rng.choice(len(cov), min(400, len(cov)), replace=False)]
            cand = sorted(cand, key=lambda c: len(op.covering_tiles(kept, f, pad, P, int(c[0]), int(c[1]))))
            done = 0
            for (cy, cx) in cand:
                tl = op.covering_tiles(kept, f, pad, P, int(cy), int(cx))
                need = [k for k in tl if k not in cache]
                if done >= 3 or len(cache) + len(need) > 24:
                    break
                for (ff, oy, ox) in need:
                    win = fe.level_window(slide, pad, det["pc"], ff, oy, ox, P)
                    tasks = [(c, s) for c, (f2, s) in zip(classes, tf) if f2 == ff]
                    Fr, Er = nn.trunk(net, arch, win)
                    g = nn.gap(Er)
                    cache[(ff, oy, ox)] = {(c, s): nn.head(Fr, nn.controller(net, arch, g, c, s)) for c, s in tasks}
                ps = np.array([cache[k][(classes[ti], s_idx)][cy + pad // f - k[1], cx + pad // f - k[2]] for k in tl])
                votes = int((ps >= 0.5).sum())
                frac_ref = votes / len(tl)
                if np.abs(ps - 0.5).min() > 1e-2:
                    assert abs(float(pt[cy, cx]) - frac_ref) <= 1e-6, (S, ti, cy, cx, pt[cy, cx], frac_ref)
                    thr = arch["vthr"][s_idx] if arch.get("vthr") else 0
                    exp_m = votes >= min(thr, len(tl)) if thr else 2 * votes >= len(tl)
                    assert int(mt[cy, cx]) == int(exp_m)
                done += 1
                checked += 1
    assert checked >= 6
