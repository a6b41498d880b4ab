"""Compute the output-logit calibration constants (head_alpha, head_beta) of the
seeded weights (SURVEY.md §8(c) O7 "logit calibration").

Calls only oracle/ and the input generators. z' = alpha z + beta with
alpha = 2 / std(z) over the calibration tiles and beta = -4 - alpha * median(z) on
a uniform pad-colour tile, so that std(z') = 2 and background z' = -4. The
printed constants are pasted into omniseg_inputs/arch.py (CALIBRATION) and cited
there; re-run whenever the architecture or the weight seed changes.

    python scripts/calibrate_head.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from omniseg_inputs import arch_string, make_slide, workload  # noqa: E402
from omniseg_inputs.arch import make_weights  # noqa: E402
from oracle import frontend as fe  # noqa: E402
from oracle import net as nn  # noqa: E402
from oracle import pipeline as op  # noqa: E402


def calibrate(cfg, n_tiles):
    w = workload(cfg)
    arch = nn.parse_arch(arch_string(w.arch))
    net = nn.unpack_weights(arch, make_weights(w.arch, w.weight_seed))
    slide = make_slide(w.slide).numpy()
    tf = op.task_factors(arch, w.scales)
    f0, s0 = tf[0]
    fr = op.front_end(slide, w.pad, w.patch, w.stride, [f0])
    lv = fe.level(fr["padded"], f0)
    kept = [k for k in fr["kept"] if k[0] == f0]
    pick = [kept[i] for i in np.linspace(0, len(kept) - 1, n_tiles).astype(int)]
    zs = []
    for (_f, oy, ox) in pick:
        F, E = nn.trunk(net, arch, lv[oy:oy + w.patch, ox:ox + w.patch])
        zs.append(nn.head_logit(F, nn.controller(net, arch, nn.gap(E), w.classes[0], s0)).ravel())
    z = np.concatenate(zs)
    bg = np.broadcast_to(fr["pc"].astype(np.uint8), (w.patch, w.patch, 3)).copy()
    F, E = nn.trunk(net, arch, bg)
    zbg = np.median(nn.head_logit(F, nn.controller(net, arch, nn.gap(E), w.classes[0], s0)))
    alpha = 2.0 / z.std()
    beta = -4.0 - alpha * zbg
    return float(alpha), float(beta)


if __name__ == "__main__":
    for cfg, n in ((1, 6), (2, 3)):
        a, b = calibrate(cfg, n)
        print(f"cfg{cfg}: head_alpha={a!r} head_beta={b!r}")
