"""Oracle, network: residual U-Net trunk, GAP, controller, dynamic head (O7-O9).

TEST INFRASTRUCTURE ONLY (see oracle/frontend.py header).

float64 throughout (the paper fixes no precision; DESIGN.md §2 R9). The
network is the one BASELINE.json's north_star names -- "a residual U-Net
encoder/decoder, then a dynamic head: a controller maps the pooled bottleneck
feature plus a one-hot class and scale code to the weights of three 1x1 conv
layers ... followed by a sigmoid" -- with the concrete block structure of
SURVEY.md §8(c) O7-O9 (DESIGN.md §2 R7-R8; the paper defers the architecture to
its earlier Omni-Seg paper, §1 / P:67 §2.2, which is not in the
container). Activations are H x W x C arrays (channels last).
"""
from __future__ import annotations

import numpy as np

HEAD = 8
THETA = 153


def parse_arch(s: str) -> dict:
    """Parse the key=value arch string (';'-separated) of DESIGN.md §3."""
    d = {}
    for kv in s.split(";"):
        if not kv:
            continue
        k, v = kv.split("=")
        d[k.strip()] = v.strip()
    return dict(levels=int(d["levels"]), base=int(d["base"]), ncls=int(d["ncls"]),
                scale_codes=[int(x) for x in d["scale_codes"].split(",")],
                slide_mag=int(d["slide_mag"]), fusion=d.get("fusion", "mean"),
                fgmin=int(d.get("fgmin", 0)), maskfg=int(d.get("maskfg", 0)),
                vthr=[int(x) for x in d["vthr"].split(",")] if "vthr" in d else None)


def unpack_weights(arch: dict, blob: np.ndarray) -> dict:
    """Blob order of SURVEY O7 / DESIGN.md §3: stem; per level l: enc RB (a, b),
    down_l (l < L-1); for l = L-2..0: up_l (1x1), dec RB (a, b); precls; Wc; bc.
    Conv weights [C_out][kh][kw][C_in] then bias [C_out]."""
    L, c0 = arch["levels"], arch["base"]
    C = [c0 << l for l in range(L)]
    blob = np.asarray(blob, dtype=np.float64)
    pos = [0]
    net = {}

    def take(shape):
        n = int(np.prod(shape))
        a = blob[pos[0]:pos[0] + n].reshape(shape)
        pos[0] += n
        return a

    def conv(name, cout, k, cin):
        net[name] = (take((cout, k, k, cin)), take((cout,)))

    conv("stem", C[0], 3, 3)
    for l in range(L):
        conv(f"enc{l}.a", C[l], 3, C[l])
        conv(f"enc{l}.b", C[l], 3, C[l])
        if l < L - 1:
            conv(f"down{l}", C[l + 1], 3, C[l])
    for l in range(L - 2, -1, -1):
        conv(f"up{l}", C[l], 1, C[l + 1])
        conv(f"dec{l}.a", C[l], 3, C[l])
        conv(f"dec{l}.b", C[l], 3, C[l])
    conv("precls", HEAD, 1, C[0])
    nin = C[L - 1] + arch["ncls"] + len(arch["scale_codes"])
    net["ctrl"] = (take((THETA, nin)), take((THETA,)))
    if pos[0] != blob.size:
        raise ValueError(f"weight blob has {blob.size} values, arch needs {pos[0]}")
    return net


def conv2d(x: np.ndarray, w: np.ndarray, b: np.ndarray, stride: int = 1) -> np.ndarray:
    """Cross-correlation with zero 'same' padding (k-1)/2 and the given stride:
    y[i, j, o] = b[o] + sum_{dy, dx, c} w[o, dy, dx, c] * x[s i + dy - r, s j + dx - r, c].
    Written as im2col + one matmul (a library primitive as a step)."""
    H, W, Cin = x.shape
    Cout, k, k2, Cin2 = w.shape
    assert k == k2 and Cin == Cin2
    r = k // 2
    xp = np.pad(x, ((r, r), (r, r), (0, 0)))
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    cols = np.empty((Ho, Wo, k, k, Cin), dtype=np.float64)
    for dy in range(k):
        for dx in range(k):
            cols[:, :, dy, dx, :] = xp[dy:dy + stride * (Ho - 1) + 1:stride,
                                       dx:dx + stride * (Wo - 1) + 1:stride, :]
    y = cols.reshape(Ho * Wo, k * k * Cin) @ w.reshape(Cout, k * k * Cin).T
    return (y + b).reshape(Ho, Wo, Cout)


def relu(x):
    return np.maximum(x, 0.0)


def up2(x):
    """Nearest-neighbour upsampling x2."""
    return x.repeat(2, axis=0).repeat(2, axis=1)


def res_block(net, name, x):
    """RB(x) = ReLU(x + conv_b(ReLU(conv_a(x))))."""
    h = relu(conv2d(x, *net[name + ".a"]))
    return relu(x + conv2d(h, *net[name + ".b"]))


def trunk(net: dict, arch: dict, tile_u8: np.ndarray):
    """Residual U-Net on one P x P x 3 u8 window.

    x = float(u8) (input scale folded into the stem); h = ReLU(stem(x));
    for l < L: E_l = RB_l(h); h = ReLU(down_l(E_l)) if l < L-1.
    D_{L-1} = E_{L-1}; for l = L-2..0: U_l = E_l + up2(up_l(D_{l+1})), D_l = RB'_l(U_l).
    F = precls(D_0) (no activation).  Returns (F [P][P][8], E_{L-1})."""
    L = arch["levels"]
    x = tile_u8.astype(np.float64)
    h = relu(conv2d(x, *net["stem"]))
    E = []
    for l in range(L):
        e = res_block(net, f"enc{l}", h)
        E.append(e)
        if l < L - 1:
            h = relu(conv2d(e, *net[f"down{l}"], stride=2))
    D = E[L - 1]
    for l in range(L - 2, -1, -1):
        U = E[l] + up2(conv2d(D, *net[f"up{l}"]))
        D = res_block(net, f"dec{l}", U)
    F = conv2d(D, *net["precls"])
    return F, E[L - 1]


def gap(E_last: np.ndarray) -> np.ndarray:
    """Global average pool of the bottleneck over its spatial extent."""
    return E_last.mean(axis=(0, 1))


def controller(net: dict, arch: dict, g: np.ndarray, cls: int, scl: int) -> np.ndarray:
    """theta = Wc [g; onehot(cls); onehot(scl)] + bc  (north_star 'controller maps the
    pooled bottleneck feature plus a one-hot class and scale code')."""
    ec = np.zeros(arch["ncls"])
    ec[cls] = 1.0
    es = np.zeros(len(arch["scale_codes"]))
    es[scl] = 1.0
    Wc, bc = net["ctrl"]
    return Wc @ np.concatenate([g, ec, es]) + bc


def split_theta(theta: np.ndarray):
    """theta layout [W1 8x8 (out,in) | b1 8 | W2 8x8 | b2 8 | W3 1x8 | b3 1] (153)."""
    o = 0
    W1 = theta[o:o + 64].reshape(8, 8); o += 64
    b1 = theta[o:o + 8]; o += 8
    W2 = theta[o:o + 64].reshape(8, 8); o += 64
    b2 = theta[o:o + 8]; o += 8
    W3 = theta[o:o + 8].reshape(1, 8); o += 8
    b3 = theta[o:o + 1]; o += 1
    assert o == THETA
    return W1, b1, W2, b2, W3, b3


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def head_logit(F: np.ndarray, theta: np.ndarray) -> np.ndarray:
    """Dynamic head: three 1x1 convs with the generated weights, ReLU between:
    z = W3 ReLU(W2 ReLU(W1 F + b1) + b2) + b3  (north_star)."""
    W1, b1, W2, b2, W3, b3 = split_theta(theta)
    h1 = relu(F @ W1.T + b1)
    h2 = relu(h1 @ W2.T + b2)
    return (h2 @ W3.T + b3)[..., 0]


def head(F: np.ndarray, theta: np.ndarray) -> np.ndarray:
    """p = sigmoid(z)."""
    return sigmoid(head_logit(F, theta))


def predict_tile(net, arch, tile_u8, tasks):
    """tasks: list of (class index, scale index). Returns p [len(tasks)][P][P]."""
    F, E_last = trunk(net, arch, tile_u8)
    g = gap(E_last)
    return np.stack([head(F, controller(net, arch, g, c, s)) for c, s in tasks])
