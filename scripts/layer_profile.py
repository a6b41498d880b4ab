"""Per-layer conv timing (CUDA events per launch) on a bench workload.
    python scripts/layer_profile.py [cfg2] [fp16f8] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from omniseg_inputs import arch_string, geometry, render, workload  # noqa: E402
from paper_2305_14566_b200 import Omniseg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dt = sys.argv[2] if len(sys.argv) > 2 else "fp16f8"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = workload(int(cfg[3:]))
w.arch["dtype"] = dt
for kv in sys.argv[4:]:  # extra arch keys, e.g. xa=0
    k, v = kv.split("=")
    w.arch[k] = int(v) if v.lstrip("-").isdigit() else v
slide = render(geometry(w.slide), device="cuda")
h = Omniseg(arch_string(w.arch), w.weights())
n = sum(h.output_size(w.H, w.W, s) for s in w.scales)
prob = torch.empty(n, device="cuda")
mask = torch.empty(n, dtype=torch.uint8, device="cuda")
area = torch.empty(len(w.scales), dtype=torch.int64, device="cuda")


def go():
    h.segment_slide(slide, w.H, w.W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, area)


go()
h.set_profile(True)
for _ in range(steps):
    go()
p = h.profile()
L = w.arch["levels"]
names = ["stem"] + [x for l in range(L) for x in ([f"enc{l}.a", f"enc{l}.b"] + ([f"down{l}"] if l < L - 1 else []))]
names += [x for l in range(L - 2, -1, -1) for x in (f"up{l}", f"dec{l}.a", f"dec{l}.b")]
tot = p["ms"]
print(f"{cfg} {dt}: conv total {tot / steps:.2f} ms/step, {p['flops'] / p['ms'] / 1e9:.1f} TFLOP/s alg; "
      f"step {h.timings()[8]:.2f} ms")
for nm, (ms, fl, cnt) in zip(names, p["layers"]):
    print(f"  {nm:8s} {ms / steps:8.3f} ms/step {100 * ms / tot:5.1f}%  {fl / ms / 1e9 if ms else 0:7.1f} TF/s alg")
