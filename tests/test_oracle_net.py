"""Pins for the oracle network (O7-O9): brute-force convolution, a library
convolution (torch.nn.functional.conv2d, fp64 CPU), special weights with closed
forms, and the dynamic head with hand-set parameters."""
import math

import numpy as np
import pytest
import scipy.special
import torch
import torch.nn.functional as Fnn

from oracle import net as nn
from omniseg_inputs import arch_dict, arch_string, blob_layout, make_weights, param_count


def conv_brute(x, w, b, stride):
    """Seven nested loops, zero padding outside the image."""
    H, W, Cin = x.shape
    Cout, k, _, _ = w.shape
    r = k // 2
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    y = np.zeros((Ho, Wo, Cout))
    for i in range(Ho):
        for j in range(Wo):
            for o in range(Cout):
                acc = b[o]
                for dy in range(k):
                    for dx in range(k):
                        yy, xx = stride * i + dy - r, stride * j + dx - r
                        if 0 <= yy < H and 0 <= xx < W:
                            for c in range(Cin):
                                acc += w[o, dy, dx, c] * x[yy, xx, c]
                y[i, j, o] = acc
    return y


@pytest.mark.parametrize("k,stride,shape", [(3, 1, (5, 7, 3)), (3, 2, (6, 8, 2)), (3, 2, (7, 5, 3)),
                                            (1, 1, (4, 6, 5)), (3, 1, (1, 1, 2))])
def test_conv_brute_force(k, stride, shape):
    rng = np.random.default_rng(k * 10 + stride)
    x = rng.standard_normal(shape)
    w = rng.standard_normal((4, k, k, shape[2]))
    b = rng.standard_normal(4)
    np.testing.assert_allclose(nn.conv2d(x, w, b, stride), conv_brute(x, w, b, stride), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("stride", [1, 2])
def test_conv_vs_torch(stride):
    rng = np.random.default_rng(stride)
    x = rng.standard_normal((16, 12, 8))
    w = rng.standard_normal((6, 3, 3, 8))
    b = rng.standard_normal(6)
    ref = Fnn.conv2d(torch.from_numpy(x).permute(2, 0, 1)[None], torch.from_numpy(w).permute(0, 3, 1, 2),
                     torch.from_numpy(b), stride=stride, padding=1)[0].permute(1, 2, 0).numpy()
    np.testing.assert_allclose(nn.conv2d(x, w, b, stride), ref, rtol=1e-12, atol=1e-12)


def test_stride2_is_subsampled_stride1():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((10, 14, 3))
    w = rng.standard_normal((5, 3, 3, 3))
    b = rng.standard_normal(5)
    np.testing.assert_allclose(nn.conv2d(x, w, b, 2), nn.conv2d(x, w, b, 1)[::2, ::2], rtol=1e-12, atol=1e-12)


def test_up2_nearest():
    x = np.arange(6.0).reshape(2, 3, 1)
    u = nn.up2(x)
    assert u.shape == (4, 6, 1)
    for i in range(4):
        for j in range(6):
            assert u[i, j, 0] == x[i // 2, j // 2, 0]


def _torch_trunk(net, arch, tile):
    """Independent re-statement of SURVEY O8 with torch primitives (NCHW, fp64)."""
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731

    def conv(x, name, stride=1):
        w, b = net[name]
        k = w.shape[1]
        return Fnn.conv2d(x, t(w).permute(0, 3, 1, 2), t(b), stride=stride, padding=k // 2)

    def rb(x, name):
        return torch.relu(x + conv(torch.relu(conv(x, name + ".a")), name + ".b"))

    L = arch["levels"]
    x = t(tile.astype(np.float64)).permute(2, 0, 1)[None]
    h = torch.relu(conv(x, "stem"))
    E = []
    for l in range(L):
        e = rb(h, f"enc{l}")
        E.append(e)
        if l < L - 1:
            h = torch.relu(conv(e, f"down{l}", 2))
    D = E[-1]
    for l in range(L - 2, -1, -1):
        U = E[l] + Fnn.interpolate(conv(D, f"up{l}"), scale_factor=2, mode="nearest")
        D = rb(U, f"dec{l}")
    F = conv(D, "precls")
    return F[0].permute(1, 2, 0).numpy(), E[-1][0].permute(1, 2, 0).numpy()


def test_trunk_vs_torch():
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    arch = nn.parse_arch(arch_string(a))
    net = nn.unpack_weights(arch, make_weights(a, 1))
    rng = np.random.default_rng(0)
    tile = rng.integers(0, 256, (32, 32, 3)).astype(np.uint8)
    F, E = nn.trunk(net, arch, tile)
    F2, E2 = _torch_trunk(net, arch, tile)
    np.testing.assert_allclose(F, F2, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(E, E2, rtol=1e-9, atol=1e-9)
    assert F.shape == (32, 32, 8) and E.shape == (8, 8, 32)


def test_param_counts_and_blob_roundtrip():
    tiny = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    big = arch_dict(levels=5, base=32, ncls=6)
    # 42,235 (tiny) / 9,678,395 (config 2+)
    assert param_count(tiny) == 42235 and param_count(big) == 9678395
    blob = make_weights(tiny, 1)
    net = nn.unpack_weights(nn.parse_arch(arch_string(tiny)), blob)
    assert net["stem"][0].shape == (8, 3, 3, 3) and net["ctrl"][0].shape == (153, 34)
    with pytest.raises(ValueError):
        nn.unpack_weights(nn.parse_arch(arch_string(tiny)), blob[:-1])
    # every conv weight exactly representable in fp16 and bf16
    for name, _ in blob_layout(tiny):
        if name.endswith(".w") and not name.startswith("ctrl"):
            w = net[name[:-2]][0]
            assert (torch.from_numpy(w).to(torch.float16).double().numpy() == w).all()
            assert (torch.from_numpy(w).to(torch.bfloat16).double().numpy() == w).all()


def test_constant_network_closed_form():
    """All conv weights zero, biases set: every layer is constant, so is F; with
    b_stem = s, every RB returns ReLU(x + b), downs give ReLU(b_down), ...; the
    final F = b_precls exactly (precls weights are zero)."""
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    arch = nn.parse_arch(arch_string(a))
    net = nn.unpack_weights(arch, np.zeros(param_count(a)))
    net["precls"] = (net["precls"][0], np.arange(8.0) - 3.0)
    net["enc2.b"] = (net["enc2.b"][0], np.full(32, 2.0))
    tile = np.random.default_rng(1).integers(0, 256, (16, 16, 3)).astype(np.uint8)
    F, E = nn.trunk(net, arch, tile)
    assert (F == (np.arange(8.0) - 3.0)).all()
    # bottleneck: E2 = ReLU(h + conv_b(.)) = ReLU(0 + 2) = 2
    assert (E == 2.0).all() and (nn.gap(E) == 2.0).all()


def test_head_hand_set_theta():
    """W1 = I, b1 = 0, W2 = I, b2 = -1, W3 = ones, b3 = 0.5:
    z = sum_i ReLU(ReLU(F_i) - 1) + 0.5."""
    theta = np.concatenate([np.eye(8).ravel(), np.zeros(8), np.eye(8).ravel(), -np.ones(8),
                            np.ones(8), [0.5]])
    rng = np.random.default_rng(3)
    F = rng.standard_normal((5, 4, 8)) * 3
    z = nn.head_logit(F, theta)
    exp = np.maximum(np.maximum(F, 0) - 1, 0).sum(-1) + 0.5
    np.testing.assert_allclose(z, exp, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(nn.head(F, theta), scipy.special.expit(exp), rtol=1e-13, atol=1e-15)


def test_controller_selects_inputs():
    """With Wc = [I | 0] selecting g and the one-hots, theta is the concatenation."""
    arch = dict(levels=3, base=8, ncls=2, scale_codes=[5, 10, 40], slide_mag=40)
    nin = 32 + 2 + 3
    Wc = np.zeros((153, nin))
    Wc[:nin, :nin] = np.eye(nin)
    bc = np.full(153, 0.25)
    net = {"ctrl": (Wc, bc)}
    g = np.arange(32.0)
    th = nn.controller(net, arch, g, 1, 2)
    exp = np.full(153, 0.25)
    exp[:32] += g
    exp[32 + 1] += 1
    exp[34 + 2] += 1
    np.testing.assert_array_equal(th, exp)


def test_sigmoid_matches_library():
    z = np.linspace(-30, 30, 1001)
    np.testing.assert_allclose(nn.sigmoid(z), scipy.special.expit(z), rtol=1e-14, atol=1e-300)
    assert nn.sigmoid(0.0) == 0.5 and math.isclose(nn.sigmoid(math.log(3)), 0.75)


def test_shift_identity_network_closed_form():
    """A network of single-tap identity convolutions with known offsets: the whole trunk
    reduces to a per-pixel formula, which pins the spatial bookkeeping end to end --
    cross-correlation orientation (not a flipped kernel), zero 'same' padding, the pixel a
    stride-2 conv samples, nearest up x2, the skip order, the residual form and the
    [C_out][kh][kw][C_in] layout. With y[i, j] = x[i-1, j] (0 on row 0; stem tap kh=0, kw=1),
    enc0 = RB with conv_a = I, conv_b = I/2 (so E0 = 1.5 y), down0 tap (kh=1, kw=2) and
    down1 centre tap, identity up-convs and identity-free decoder RBs:
        F[i, j, c] = 1.5 (y[i, j] + y[2(i//2), 2(j//2) + 1] + y[4(i//4), 4(j//4) + 1])
    for c < 3 (channel c of the input), and GAP(E2) = 1.5 mean_{i,j} y[4i, 4j+1]."""
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    arch = nn.parse_arch(arch_string(a))
    net = nn.unpack_weights(arch, np.zeros(param_count(a)))

    def tap(name, kh, kw, scale=1.0):
        w, b = net[name]
        w = np.zeros_like(w)
        for c in range(3):
            w[c, kh, kw, c] = scale
        net[name] = (w, b)

    tap("stem", 0, 1)
    tap("enc0.a", 1, 1)
    tap("enc0.b", 1, 1, 0.5)
    tap("down0", 1, 2)
    tap("down1", 1, 1)
    tap("up1", 0, 0)
    tap("up0", 0, 0)
    tap("precls", 0, 0)
    P = 16
    x = np.random.default_rng(7).integers(0, 256, (P, P, 3)).astype(np.uint8)
    y = np.zeros((P, P, 3))
    y[1:] = x[:-1]
    F, E = nn.trunk(net, arch, x)
    exp = np.zeros((P, P, 3))
    for i in range(P):
        for j in range(P):
            exp[i, j] = 1.5 * (y[i, j] + y[2 * (i // 2), 2 * (j // 2) + 1] + y[4 * (i // 4), 4 * (j // 4) + 1])
    assert (F[:, :, :3] == exp).all()
    assert (F[:, :, 3:] == 0).all()
    np.testing.assert_allclose(nn.gap(E)[:3], 1.5 * y[0::4, 1::4].mean(axis=(0, 1)), rtol=1e-14)
