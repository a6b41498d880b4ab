"""Time omniseg_render_overlay on the cfg4 slide with device-resident buffers
(CUDA events) and report its HBM throughput against the algorithmic bytes
(slide 3 B/px + masks + 40x out 3 B/px + 10x out 3/16 B/px).
    python scripts/overlay_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from omniseg_inputs import arch_string, geometry, render, workload  # noqa: E402
from paper_2305_14566_b200 import Omniseg  # noqa: E402

w = workload(4)
H, W = w.H, w.W
slide = render(geometry(w.slide), device="cuda", chunk_rows=2048)
h = Omniseg(arch_string(w.arch), w.weights())
sizes = [h.output_size(H, W, s) for s in w.scales]
prob = torch.empty(sum(sizes), dtype=torch.float32, device="cuda")
mask = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
h.segment_slide(slide, H, W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, None)
out40 = torch.empty((H, W, 3), dtype=torch.uint8, device="cuda")
out10 = torch.empty(((H + 3) // 4, (W + 3) // 4, 3), dtype=torch.uint8, device="cuda")
for _ in range(2):
    h.render_overlay(slide, H, W, mask, w.scales, w.classes, out40, out10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    h.render_overlay(slide, H, W, mask, w.scales, w.classes, out40, out10)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = H * W * 3 * 2 + sum(sizes) + out10.numel()
print(f"render_overlay cfg4 {H}x{W}, {len(w.scales)} tasks: {ms:.2f} ms, algorithmic {alg / 1e9:.2f} GB -> "
      f"{alg / ms / 1e6:.0f} GB/s (includes the call's stream sync)")
