"""Special-weight networks with closed-form outputs (test infrastructure).

They build weight BLOBS in the documented order (omniseg_inputs.arch.blob_layout), so the
same network runs through the oracle (oracle.net.unpack_weights) and through the C ABI.
Their closed forms are restated here from the network definition (SURVEY §8(c) O8/O9,
DESIGN.md R9), not from either implementation.

* shift-identity network: single-tap identity convolutions at known offsets; the trunk
  reduces to F[i, j, c] = 1.5 (y[i, j] + sum_{l=1}^{L-1} y[2^l (i >> l), 2^l (j >> l) + 1]),
  c < 3, with y = the window shifted down one row (0 on row 0) -- pins tap orientation,
  zero 'same' padding, the stride-2 sample, nearest up x2, skips and the weight layout.
* probe network: centre-tap identity stem, every other conv zero: F = the window itself
  (channels 0..2), so p at a slide pixel does not depend on WHICH window covers it --
  the stitched canvas is a closed form of the level image (pins window gather, the
  pyramid level a scale reads and the canvas placement at every level factor f).
"""
from __future__ import annotations

import numpy as np

from omniseg_inputs.arch import arch_dict, arch_string, blob_layout, param_count
from oracle import net as nn


def _blob(a, net):
    blob = np.concatenate([net[n.rsplit(".", 1)[0]][0 if n.endswith(".w") else 1].ravel()
                           for n, _ in blob_layout(a)]).astype(np.float32)
    assert blob.size == param_count(a)
    return blob


def _zero_net(levels, base, ncls, scale_codes, slide_mag, dtype, batch):
    a = arch_dict(levels=levels, base=base, ncls=ncls, scale_codes=scale_codes, slide_mag=slide_mag, batch=batch)
    a["dtype"] = dtype
    arch = nn.parse_arch(arch_string(a))
    return a, nn.unpack_weights(arch, np.zeros(param_count(a)))


def _tap(net, name, kh, kw, scale=1.0):
    w = np.zeros_like(net[name][0])
    for c in range(3):
        w[c, kh, kw, c] = scale
    net[name] = (w, net[name][1])


def head_theta(w3: float, b3: float, ch: int = 0) -> np.ndarray:
    """theta (layout W1 8x8 | b1 | W2 8x8 | b2 | W3 1x8 | b3) with W1 = W2 = I,
    b1 = b2 = 0, W3 = w3 e_ch: z = w3 ReLU(ReLU(F_ch)) + b3."""
    theta = np.zeros(153)
    theta[0:64] = np.eye(8).ravel()
    theta[72:136] = np.eye(8).ravel()
    theta[144 + ch] = w3
    theta[152] = b3
    return theta


def shift_identity_net(levels, base, bc=None, dtype="fp16f8", ncls=1, scale_codes=(1,), slide_mag=1, batch=16):
    """(arch dict, oracle net dict, blob) of the shift-identity network; bc: controller bias
    (= theta, the controller weights being zero)."""
    a, net = _zero_net(levels, base, ncls, scale_codes, slide_mag, dtype, batch)
    for name, kh, kw, s in (("stem", 0, 1, 1.0), ("enc0.a", 1, 1, 1.0), ("enc0.b", 1, 1, 0.5), ("down0", 1, 2, 1.0),
                            ("precls", 0, 0, 1.0)):
        _tap(net, name, kh, kw, s)
    for l in range(1, levels - 1):
        _tap(net, f"down{l}", 1, 1)
    for l in range(levels - 1):
        _tap(net, f"up{l}", 0, 0)
    if bc is not None:
        net["ctrl"] = (net["ctrl"][0], np.asarray(bc, np.float64))
    return a, net, _blob(a, net)


def shift_identity_F(tile: np.ndarray, levels: int) -> np.ndarray:
    """Closed form of the shift-identity trunk's F[..., :3] for one window."""
    P = tile.shape[0]
    i = np.arange(P)[:, None]
    j = np.arange(P)[None, :]
    y = np.zeros((P, P, 3))
    y[1:] = tile[:-1]
    exp = y.copy()
    for l in range(1, levels):
        exp += y[(i >> l) << l, ((j >> l) << l) + 1]
    return 1.5 * exp


def probe_net(levels, base, bc, dtype="fp16f8", ncls=1, scale_codes=(1,), slide_mag=1, batch=16):
    """(arch dict, oracle net dict, blob) of the probe network: stem = centre-tap identity,
    precls = identity on channels 0..2, every other conv and bias zero, controller weights
    zero and bias `bc`. Every residual block then returns its input, every down / deeper
    level is 0 and every up-add adds 0, so F = window (channels 0..2) and GAP = 0."""
    a, net = _zero_net(levels, base, ncls, scale_codes, slide_mag, dtype, batch)
    _tap(net, "stem", 1, 1)
    _tap(net, "precls", 0, 0)
    net["ctrl"] = (net["ctrl"][0], np.asarray(bc, np.float64))
    return a, net, _blob(a, net)


def block_mean_brute(padded: np.ndarray, f: int, rows=None) -> np.ndarray:
    """Area mean over f x f blocks rounded half up, by explicit summation of the f^2 shifted
    sub-grids (a restatement independent of oracle.frontend.level's reshape)."""
    Hp, Wp, C = padded.shape
    acc = np.zeros((Hp // f, Wp // f, C), np.int64)
    for dy in range(f):
        for dx in range(f):
            acc += padded[dy::f, dx::f].astype(np.int64)
    return ((2 * acc + f * f) // (2 * f * f)).astype(np.uint8)
