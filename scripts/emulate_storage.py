"""Diagnostic (not the oracle, not a test): the oracle network re-run with 16-bit
rounding at the GPU path's storage points, to separate kernel bugs from the
numerics of 16-bit activations.
    python scripts/emulate_storage.py [cfg] [n] [fp16|bf16]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from omniseg_inputs import arch_string, make_slide, workload  # noqa: E402
from oracle import net as nn  # noqa: E402
from oracle import pipeline as op  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dt = sys.argv[3] if len(sys.argv) > 3 else "fp16"
tdt = torch.float16 if dt == "fp16" else torch.bfloat16


def q(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(tdt).double().numpy()


def trunk_q(net, arch, tile):
    L = arch["levels"]
    conv = lambda x, name, s=1: nn.conv2d(x, *net[name], stride=s)  # noqa: E731
    h = q(nn.relu(conv(tile.astype(np.float64), "stem")))
    E = []
    for l in range(L):
        t = q(nn.relu(conv(h, f"enc{l}.a")))
        e = q(nn.relu(h + conv(t, f"enc{l}.b")))
        E.append(e)
        if l < L - 1:
            h = q(nn.relu(conv(e, f"down{l}", 2)))
    D = E[-1]
    for l in range(L - 2, -1, -1):
        U = q(E[l] + nn.up2(conv(D, f"up{l}")))
        t = q(nn.relu(conv(U, f"dec{l}.a")))
        D = q(nn.relu(U + conv(t, f"dec{l}.b")))
    return conv(D, "precls"), E[-1]


w = workload(cfg)
arch = nn.parse_arch(arch_string(w.arch))
net = nn.unpack_weights(arch, w.weights())
slide = make_slide(w.slide).numpy()
fr = op.front_end(slide, w.pad, w.patch, w.stride, [1])
kept = fr["kept"]
pick = [kept[i] for i in np.linspace(0, len(kept) - 1, n).astype(int)]
for (_, oy, ox) in pick:
    tile = fr["padded"][oy:oy + w.patch, ox:ox + w.patch]
    Fr, Er = nn.trunk(net, arch, tile)
    Fq, Eq = trunk_q(net, arch, tile)
    th = nn.controller(net, arch, nn.gap(Er), w.classes[0], 0)
    zr = nn.head_logit(Fr, th)
    zq = nn.head_logit(Fq, th)
    d = np.abs(nn.sigmoid(zq) - nn.sigmoid(zr))
    dF = np.abs(Fq - Fr)
    print(f"{(oy, ox)}: dF max rel {dF.max() / np.abs(Fr).max():.3g} mean rel {dF.mean() / np.abs(Fr).mean():.3g}; "
          f"z mean {zr.mean():.3g} std {zr.std():.3g} dz max {np.abs(zq - zr).max():.3g}; dp max {d.max():.4g}")

# ---- rounding-flip proxy: storage-rounded network computed with fp32 accumulation vs fp64
print("-- fp32-accumulate + storage rounding  vs  fp64-accumulate + storage rounding")
orig = nn.conv2d


def conv32(x, wt, b, stride=1):
    return orig(x.astype(np.float32).astype(np.float64), wt, b, stride).astype(np.float32).astype(np.float64) \
        if False else _c32(x, wt, b, stride)


def _c32(x, wt, b, stride):
    H, W, Cin = x.shape
    Cout, k, _, _ = wt.shape
    r = k // 2
    xp = np.pad(x.astype(np.float32), ((r, r), (r, r), (0, 0)))
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    cols = np.empty((Ho, Wo, k, k, Cin), np.float32)
    for dy in range(k):
        for dx in range(k):
            cols[:, :, dy, dx, :] = xp[dy:dy + stride * (Ho - 1) + 1:stride, dx:dx + stride * (Wo - 1) + 1:stride, :]
    y = cols.reshape(Ho * Wo, -1)[:, ::-1] @ wt.reshape(Cout, -1).T.astype(np.float32)[::-1, :]
    return (y + b.astype(np.float32)).reshape(Ho, Wo, Cout).astype(np.float64)


for (_, oy, ox) in pick:
    tile = fr["padded"][oy:oy + w.patch, ox:ox + w.patch]
    nn.conv2d = orig
    Fq, Eq = trunk_q(net, arch, tile)
    nn.conv2d = _c32
    F32, E32 = trunk_q(net, arch, tile)
    nn.conv2d = orig
    Fr, Er = nn.trunk(net, arch, tile)
    th = nn.controller(net, arch, nn.gap(Er), w.classes[0], 0)
    d = np.abs(nn.sigmoid(nn.head_logit(F32, th)) - nn.sigmoid(nn.head_logit(Fq, th)))
    dF = np.abs(F32 - Fq)
    print(f"{(oy, ox)}: dF max rel {dF.max() / np.abs(Fq).max():.3g} frac F differing {(dF > 0).mean():.3g}; dp max {d.max():.4g}")
