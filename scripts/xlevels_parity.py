"""Numerics experiment: which U-Net levels need x2 (hi+lo) activation storage to meet
|dp| <= 1e-2 against the fp64 oracle? (R9)
    python scripts/xlevels_parity.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from omniseg_inputs import arch_string, make_slide, workload  # noqa: E402
from oracle import net as nn  # noqa: E402
from oracle import pipeline as op  # noqa: E402
from paper_2305_14566_b200 import Omniseg  # noqa: E402


def stitched(cfg, crop, xls):
    w = workload(cfg)
    slide = make_slide(w.slide).numpy()
    if crop:
        slide = slide[crop[0]:crop[1], crop[2]:crop[3]].copy()
        slide[:4, :4] = slide[-4:, -4:] * 0 + 235
    H, W = slide.shape[:2]
    t = time.time()
    ref = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes)
    print(f"cfg{cfg} crop {crop}: {len(ref['kept'])} tiles, oracle {time.time() - t:.0f}s")
    for xl in xls:
        a = dict(w.arch)
        if isinstance(xl, str):
            for kv in xl.split("+"):  # several keys: k1=v1+k2=v2
                k, v = kv.split("=")
                a[k] = int(v) if v.lstrip("-").isdigit() else v
        else:
            a["xlevels"] = xl
        h = Omniseg(arch_string(a), w.weights())
        n = sum(h.output_size(H, W, s) for s in w.scales)
        prob = np.zeros(n, np.float32)
        mask = np.zeros(n, np.uint8)
        h.segment_slide(slide, H, W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, None)
        o, worst, agree = 0, 0.0, 1.0
        for k, s in enumerate(w.scales):
            f = w.arch["slide_mag"] // s
            hh, ww = (H + f - 1) // f, (W + f - 1) // f
            d = np.abs(prob[o:o + hh * ww].reshape(hh, ww) - ref["prob"][k])
            worst = max(worst, d.max())
            agree = min(agree, (mask[o:o + hh * ww].reshape(hh, ww) == ref["mask"][k]).mean())
            o += hh * ww
        print(f"   xlevels={xl}: max |dp| {worst:.4g}  mask agreement {agree:.5f}  {'PASS' if worst <= 1e-2 and agree >= 0.999 else 'fail'}")


import sys as _s
if len(_s.argv) > 1:
    stitched(1, None, _s.argv[1:])
    stitched(2, (1024, 2560, 1024, 2560), _s.argv[1:])
else:
    stitched(1, None, [0, 1, 2, 3])
    stitched(2, (1024, 2560, 1024, 2560), [0, 1, 2, 3, 4, 5])
