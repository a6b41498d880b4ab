"""Diagnostic: GPU trunk/head vs oracle on a few windows, per-stage error stats.
    python scripts/diag_tiles.py [cfg] [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from omniseg_inputs import arch_string, make_slide, workload  # noqa: E402
from oracle import frontend as fe  # noqa: E402
from oracle import net as nn  # noqa: E402
from oracle import pipeline as op  # noqa: E402
from paper_2305_14566_b200 import Omniseg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = workload(cfg)
arch = nn.parse_arch(arch_string(w.arch))
net = nn.unpack_weights(arch, w.weights())
slide = make_slide(w.slide).numpy() if cfg <= 2 else None
fr = op.front_end(slide, w.pad, w.patch, w.stride, [1])
lv = fr["padded"]
kept = fr["kept"]
pick = [kept[i] for i in np.linspace(0, len(kept) - 1, n).astype(int)]
tiles = np.stack([lv[oy:oy + w.patch, ox:ox + w.patch] for (_, oy, ox) in pick])
h = Omniseg(arch_string(w.arch), w.weights())
tf = op.task_factors(arch, w.scales)
tasks = [(c, s) for c, (f, s) in zip(w.classes, tf)]
Cb = arch["base"] << (arch["levels"] - 1)
p, F, g = h.predict_tiles(tiles, tasks, with_F=True, with_g=True, c_bottleneck=Cb)
for i in range(n):
    Fr, Er = nn.trunk(net, arch, tiles[i])
    gr = nn.gap(Er)
    dF = np.abs(F[i] - Fr)
    print(f"tile {i} {pick[i]}: |F| max {np.abs(Fr).max():.3g}  dF max {dF.max():.3g} "
          f"(rel {dF.max() / np.abs(Fr).max():.3g}) at {np.unravel_index(dF.argmax(), dF.shape)}  "
          f"mean rel {dF.mean() / np.abs(Fr).mean():.3g}")
    print(f"   g: max {np.abs(gr).max():.3g} dg max {np.abs(g[i] - gr).max():.3g}")
    for k, (c, s) in enumerate(tasks):
        th = nn.controller(net, arch, gr, c, s)
        zr = nn.head_logit(Fr, th)
        pr = nn.sigmoid(zr)
        d = np.abs(p[i, k] - pr)
        yx = np.unravel_index(d.argmax(), d.shape)
        print(f"   task {k}: dp max {d.max():.4g} at {yx} (p_ref {pr[yx]:.4f}, z_ref {zr[yx]:.3f}), "
              f"p99.9 {np.quantile(d, 0.999):.3g}, frac>1e-2 {(d > 1e-2).mean():.4f}")
