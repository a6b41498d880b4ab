"""Seeded synthetic whole-slide images shaped like the paper's workloads.

INPUT GENERATOR ONLY (no arithmetic of the method lives here). Both the oracle
side and the CUDA side consume these slides; neither side's code is used here.

The paper's workload is KPMP kidney needle-biopsy WSIs at 40x, 0.25 um/px
(§3.1, §4); those files are not in the container and
are NOT reproduced. The stand-ins follow BASELINE.json configs[0..4] and the
recipe of SURVEY.md §8(d) (restated in DESIGN.md §4):

* every pixel value comes from a counter-based integer hash of (seed, y, x, c),
  so any window of any slide regenerates bit-identically on CPU or GPU;
* geometry (ellipses, cores, random field) is drawn on the host with
  ``numpy.random.default_rng(seed)`` and evaluated with integer or
  separately-rounded float64 operations only (no transcendental per pixel);
* labels: 0 background 235+-5, 1 tissue (200,120,170)+-20, 2 tubule wall
  (160,80,140)+-10, 3 lumen (225,205,220)+-5, 4 nucleus (90,60,140)+-10;
* the top-left 4x4 corner is always background, so the paper's pad colour
  (mean of the top-left 2x2) equals the background.
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import torch

M32 = 0xFFFFFFFF
BASE = ((235, 235, 235), (200, 120, 170), (160, 80, 140), (225, 205, 220), (90, 60, 140))
AMP = (5, 20, 10, 5, 10)
RING_CELL = 160
NUC_CELL = 40
FIELD_STEP = 64


def _h32(x: torch.Tensor) -> torch.Tensor:
    # xorshift-multiply finaliser; every product stays below 2^63 (constants < 2^31).
    x = x & M32
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & M32
    x = x ^ (x >> 15)
    x = (x * 0x2C1B3C6D) & M32
    x = x ^ (x >> 16)
    return x


def _hash2(a: torch.Tensor, b: torch.Tensor, salt: int) -> torch.Tensor:
    return _h32(_h32((a & M32) ^ (salt & M32)) ^ (b & M32))


# --------------------------------------------------------------------------
# geometry (host side, numpy RNG)
# --------------------------------------------------------------------------
def _ellipse_params(rng, W, H, axes):
    a = float(rng.uniform(*axes))
    b = float(rng.uniform(*axes))
    th = float(rng.uniform(0.0, math.pi))
    cx = float(rng.uniform(0, W))
    cy = float(rng.uniform(0, H))
    c, s = math.cos(th), math.sin(th)
    # (u/a)^2 + (v/b)^2 <= 1 with u = dx c + dy s, v = -dx s + dy c
    # -> A dx^2 + B dx dy + C dy^2 <= 1
    A = c * c / (a * a) + s * s / (b * b)
    B = 2.0 * c * s * (1.0 / (a * a) - 1.0 / (b * b))
    C = s * s / (a * a) + c * c / (b * b)
    r = max(a, b)
    return (cx, cy, A, B, C, r)


def _coverage_grid(ells, W, H, step=32):
    ys = np.arange(step // 2, H, step, dtype=np.float64)[:, None]
    xs = np.arange(step // 2, W, step, dtype=np.float64)[None, :]
    m = np.zeros((ys.shape[0], xs.shape[1]), bool)
    for (cx, cy, A, B, C, r) in ells:
        dx = xs - cx
        dy = ys - cy
        m |= (A * dx * dx + B * dx * dy + C * dy * dy) <= 1.0
    return m


def geometry(spec: dict) -> dict:
    """Host-side shape parameters for a slide spec (deterministic in spec['seed'])."""
    rng = np.random.default_rng(spec["seed"])
    W, H = spec["W"], spec["H"]
    g = dict(kind=spec["kind"], W=W, H=H, seed=spec["seed"],
             rings=spec.get("rings", False), nuclei=spec.get("nuclei", False))
    if spec["kind"] == "blobs":
        ells = []
        if spec.get("coverage"):
            while True:
                for _ in range(8):
                    ells.append(_ellipse_params(rng, W, H, spec["axes"]))
                if _coverage_grid(ells, W, H).mean() >= spec["coverage"]:
                    break
        else:
            for _ in range(spec["n_blobs"]):
                ells.append(_ellipse_params(rng, W, H, spec["axes"]))
        g["ellipses"] = ells
    elif spec["kind"] == "cores":
        n = spec["n_cores"]
        y = np.arange(H, dtype=np.float64)
        cores = []
        for i in range(n):
            width = float(rng.uniform(3000, 3600))
            amp = float(rng.uniform(300, 1100))
            lam = float(rng.uniform(H / 3.0, H))
            ph = float(rng.uniform(0, 2 * math.pi))
            x0 = W * (i + 0.5) / n + float(rng.uniform(-200, 200))
            y0, y1 = int(0.02 * H), int(0.98 * H)
            xc = np.rint(x0 + amp * np.sin(2 * math.pi * y / lam + ph)).astype(np.int64)
            cores.append(dict(xc=xc, hw=int(width // 2), y0=y0, y1=y1))
        g["cores"] = cores
    elif spec["kind"] == "field":
        gh = H // FIELD_STEP + 2
        gw = W // FIELD_STEP + 2
        yy = np.arange(gh, dtype=np.float64)[:, None] * FIELD_STEP
        xx = np.arange(gw, dtype=np.float64)[None, :] * FIELD_STEP
        f = np.zeros((gh, gw))
        for _ in range(24):
            lam = float(rng.uniform(2500, 12000))
            th = float(rng.uniform(0, 2 * math.pi))
            ph = float(rng.uniform(0, 2 * math.pi))
            f += np.cos(2 * math.pi * (xx * math.cos(th) + yy * math.sin(th)) / lam + ph)
        fi = np.rint(f * 1000).astype(np.int64)
        # threshold at the quantile giving the requested tissue fraction, measured on
        # the same integer bilinear interpolation the renderer uses, every 16 px
        sub = _field_eval_np(fi, np.arange(8, H, 16)[:, None], np.arange(8, W, 16)[None, :])
        tau = int(np.quantile(sub, 1.0 - spec["fraction"]))
        g["field"] = fi
        g["tau"] = tau
    else:
        raise ValueError(spec["kind"])
    return g


def _field_eval_np(fi, y, x):
    i, fy = y // FIELD_STEP, y % FIELD_STEP
    j, fx = x // FIELD_STEP, x % FIELD_STEP
    top = fi[i, j] * (FIELD_STEP - fx) + fi[i, j + 1] * fx
    bot = fi[i + 1, j] * (FIELD_STEP - fx) + fi[i + 1, j + 1] * fx
    return top * (FIELD_STEP - fy) + bot * fy


# --------------------------------------------------------------------------
# rendering (torch; identical integer results on CPU and CUDA)
# --------------------------------------------------------------------------
def _labels(g, y, x, dev):
    """Label map for the window rows y[:,0], cols x[0,:] (int64 tensors)."""
    h, w = y.shape[0], x.shape[1]
    lab = torch.zeros((h, w), dtype=torch.uint8, device=dev)
    if g["kind"] == "blobs":
        yf = y.to(torch.float64)
        xf = x.to(torch.float64)
        y0, y1 = int(y[0, 0]), int(y[-1, 0])
        x0, x1 = int(x[0, 0]), int(x[0, -1])
        for (cx, cy, A, B, C, r) in g["ellipses"]:
            if cy + r < y0 or cy - r > y1 or cx + r < x0 or cx - r > x1:
                continue
            dx = xf - cx
            dy = yf - cy
            q = torch.mul(torch.mul(dx, dx), A)
            q = torch.add(q, torch.mul(torch.mul(dx, dy), B))
            q = torch.add(q, torch.mul(torch.mul(dy, dy), C))
            lab[q <= 1.0] = 1
    elif g["kind"] == "cores":
        yi = y[:, 0]
        for c in g["cores"]:
            xc = torch.as_tensor(c["xc"], device=dev)[yi.clamp(0, g["H"] - 1)][:, None]
            inside = (x - xc).abs() <= c["hw"]
            inrow = ((y >= c["y0"]) & (y < c["y1"]))
            # rounded ends: disc of radius hw around the end-row centres
            body = inside & inrow
            for ye in (c["y0"], c["y1"] - 1):
                xe = int(c["xc"][ye])
                d2 = (x - xe) * (x - xe) + (y - ye) * (y - ye)
                body = body | (d2 <= c["hw"] * c["hw"])
            lab[body] = 1
    elif g["kind"] == "field":
        fi = torch.as_tensor(g["field"], device=dev)
        i, fy = y // FIELD_STEP, y % FIELD_STEP
        j, fx = x // FIELD_STEP, x % FIELD_STEP
        gw = fi.shape[1]
        flat = fi.reshape(-1)
        top = flat[i * gw + j] * (FIELD_STEP - fx) + flat[i * gw + j + 1] * fx
        bot = flat[(i + 1) * gw + j] * (FIELD_STEP - fx) + flat[(i + 1) * gw + j + 1] * fx
        val = top * (FIELD_STEP - fy) + bot * fy
        lab[val > g["tau"]] = 1
    seed = g["seed"]
    if g["rings"]:
        ci, cj = y // RING_CELL, x // RING_CELL
        hh = _hash2(ci, cj, seed * 7919 + 11)
        present = (hh % 100) < 60
        cy = ci * RING_CELL + RING_CELL // 2 + (hh >> 8) % 31 - 15
        cx = cj * RING_CELL + RING_CELL // 2 + (hh >> 13) % 31 - 15
        rout = 20 + (hh >> 18) % 41
        wall = 8 + (hh >> 24) % 8
        d2 = (y - cy) * (y - cy) + (x - cx) * (x - cx)
        tissue = lab == 1
        inwall = present & tissue & (d2 <= rout * rout) & (d2 > (rout - wall) * (rout - wall))
        inlum = present & tissue & (d2 <= (rout - wall) * (rout - wall))
        lab[inwall] = 2
        lab[inlum] = 3
    if g["nuclei"]:
        ci, cj = y // NUC_CELL, x // NUC_CELL
        hh = _hash2(ci, cj, seed * 104729 + 17)
        present = (hh % 100) < 35
        cy = ci * NUC_CELL + NUC_CELL // 2 + (hh >> 8) % 25 - 12
        cx = cj * NUC_CELL + NUC_CELL // 2 + (hh >> 13) % 25 - 12
        r = 3 + (hh >> 18) % 4
        d2 = (y - cy) * (y - cy) + (x - cx) * (x - cx)
        lab[present & (lab == 1) & (d2 <= r * r)] = 4
    lab[(y < 4) & (x < 4)] = 0
    return lab


def render(g: dict, r0: int = 0, r1: int | None = None, c0: int = 0, c1: int | None = None,
           device="cpu", chunk_rows: int = 1024) -> torch.Tensor:
    """uint8 [r1-r0][c1-c0][3] window of the slide described by geometry ``g``."""
    H, W = g["H"], g["W"]
    r1 = H if r1 is None else r1
    c1 = W if c1 is None else c1
    assert 0 <= r0 <= r1 <= H and 0 <= c0 <= c1 <= W
    dev = torch.device(device)
    out = torch.empty((r1 - r0, c1 - c0, 3), dtype=torch.uint8, device=dev)
    base = torch.tensor(BASE, dtype=torch.int64, device=dev)
    amp = torch.tensor(AMP, dtype=torch.int64, device=dev)
    x = torch.arange(c0, c1, dtype=torch.int64, device=dev)[None, :]
    for a in range(r0, r1, chunk_rows):
        b = min(r1, a + chunk_rows)
        y = torch.arange(a, b, dtype=torch.int64, device=dev)[:, None]
        lab = _labels(g, y, x, dev).to(torch.int64)
        key = y * W + x                                  # < 2^31 for all configs
        am = amp[lab]
        for c in range(3):
            hsh = _hash2(key * 3 + c, key >> 31, g["seed"] * 65537 + 3)
            val = base[lab, c] + hsh % (2 * am + 1) - am
            out[a - r0:b - r0, :, c] = val.clamp(0, 255).to(torch.uint8)
    return out


def make_slide(spec: dict, device="cpu", **kw) -> torch.Tensor:
    return render(geometry(spec), device=device, **kw)


def sha256(t: torch.Tensor) -> str:
    return hashlib.sha256(t.contiguous().cpu().numpy().tobytes()).hexdigest()


def blank_slide(H: int, W: int, seed: int = 99, device="cpu") -> torch.Tensor:
    """All-background slide (the north_star's 'all-background slides yield empty masks')."""
    g = dict(kind="blobs", W=W, H=H, seed=seed, rings=False, nuclei=False, ellipses=[])
    return render(g, device=device)


def random_tiles(n: int, P: int, seed: int, device="cpu") -> torch.Tensor:
    """n x P x P x 3 uint8 tiles cut from a seeded blob slide (tile-level parity inputs)."""
    spec = dict(kind="blobs", seed=seed, W=P * 4, H=P * max(1, n), n_blobs=6 * max(1, n),
                axes=(P // 8, P // 2), rings=True, nuclei=True)
    s = make_slide(spec, device=device)
    return torch.stack([s[i * P:(i + 1) * P, (i % 3) * P:(i % 3) * P + P] for i in range(n)])
