"""Small end-to-end workload for compute-sanitizer (memcheck / synccheck / racecheck / initcheck):
the config-1 tiny network on a 512^2 crop through every product kernel family -- pyramid,
detection, tile selection, fused gather + stem, the tcgen05 conv kernels, GAP + controller,
fused head + stitch, finalize -- plus the vote / fgmin / maskfg paths (union-find) and the
overlay; and one 256^2-window pass of the bench network (levels 5, base 32) so the
32-channel stem, no-swizzle, stride-2 and per-tap kernels run too.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from omniseg_inputs import arch_string, make_slide, workload  # noqa: E402
from paper_2305_14566_b200 import Omniseg  # noqa: E402


def run(arch, blob, slide, pad, P, S, scales, classes):
    h = Omniseg(arch_string(arch), blob)
    H, W = slide.shape[:2]
    n = sum(h.output_size(H, W, s) for s in scales)
    prob = torch.zeros(n, dtype=torch.float32, device="cuda")
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    area = torch.zeros(len(scales), dtype=torch.int64, device="cuda")
    d = torch.from_numpy(slide).cuda()
    h.segment_slide(d, H, W, pad, P, S, scales, classes, prob, mask, area)
    torch.cuda.synchronize()
    return h, prob, mask, area


def main():
    w = workload(1)
    slide = make_slide(w.slide).numpy()[:512, :512].copy()
    run(w.arch, w.weights(), slide, 64, 256, 128, w.scales, w.classes)
    a = dict(w.arch, fusion="vote", fgmin=20, maskfg=1)
    run(a, w.weights(), slide, 64, 128, 64, w.scales, w.classes)
    w3 = workload(3)
    big = make_slide(w.slide).numpy()[:1024, :1024].copy()
    a3 = dict(w3.arch, batch=8)
    h, prob, mask, area = run(a3, w3.weights(), big, 512, 256, 128, (40, 10, 5), (4, 2, 0))
    H, W = big.shape[:2]
    out40 = torch.zeros((H, W, 3), dtype=torch.uint8, device="cuda")
    out10 = torch.zeros(((H + 3) // 4, (W + 3) // 4, 3), dtype=torch.uint8, device="cuda")
    h.render_overlay(torch.from_numpy(big).cuda(), H, W, mask, (40, 10, 5), (4, 2, 0), out40, out10)
    torch.cuda.synchronize()
    print("sanitize workload done: %d tiles, area %s" % (len(h.tiles()), area.tolist()))


if __name__ == "__main__":
    main()
