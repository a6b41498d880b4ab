"""GPU parity of the tcgen05 implicit-GEMM convolution (through the C ABI,
omniseg_debug_conv) against the oracle's convolution (fp64) on seeded inputs.

Inputs and weights are drawn exactly representable in fp16, so the only
differences are the fp32 accumulation order and the final 16-bit rounding of the
stored output: |gpu - oracle| <= 2^-10 |oracle| (fp16 half-ulp, relative) + 1e-3
absolute slack for cancellation."""
import numpy as np
import pytest

from oracle import net as nn
from omniseg_inputs import arch_dict, arch_string, make_weights

pytestmark = pytest.mark.gpu

TOL_REL = 2.0 ** -10


@pytest.fixture(scope="module")
def h(gpu_lib):
    from paper_2305_14566_b200 import Omniseg
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1, batch=4)
    return Omniseg(arch_string(a), make_weights(a, 1))


def _f16(a):
    return a.astype(np.float16).astype(np.float64)


def _ref(x, w, b, stride, r, mode):
    out = []
    for i in range(x.shape[0]):
        y = nn.conv2d(x[i], w, b, stride)
        if mode == 0:
            y = np.maximum(y, 0)
        elif mode == 1:
            y = np.maximum(y + r[i], 0)
        elif mode == 2:
            y = r[i] + nn.up2(y)
        elif mode == 3 and r is not None:
            y = y + r[i]
        out.append(y)
    return np.stack(out)


CASES = [
    # B, H, W, Cin, Cout, k, stride, mode
    (2, 16, 16, 16, 16, 3, 1, 0),
    (2, 64, 64, 32, 32, 3, 1, 0),
    (1, 128, 128, 32, 32, 3, 1, 1),
    (1, 256, 256, 32, 64, 3, 2, 0),
    (2, 32, 32, 64, 64, 3, 1, 1),
    (2, 32, 32, 64, 128, 3, 2, 0),
    (1, 16, 16, 256, 256, 3, 1, 0),
    (1, 16, 16, 256, 512, 3, 1, 1),
    (1, 16, 16, 512, 512, 3, 1, 0),
    (2, 16, 16, 64, 32, 1, 1, 2),
    (1, 32, 32, 512, 256, 1, 1, 2),
    (3, 8, 16, 32, 16, 3, 1, 3),
    (1, 512, 512, 32, 32, 3, 1, 0),
    (1, 32, 32, 48, 48, 3, 1, 1),   # 48 channels: K chunk 16, N tile 16
    # multi-row 3x3 kernel (conv3_rows_kernel): N<=128, hb in {1,2}
    (1, 256, 256, 16, 16, 3, 1, 1),   # R=16
    (1, 256, 256, 64, 64, 3, 1, 0),   # R=4, BK=32
    (1, 128, 128, 128, 128, 3, 1, 1), # R=2
    (2, 64, 64, 64, 64, 3, 1, 3),     # hb=2
    (1, 4, 128, 32, 32, 3, 1, 0),     # tiles_y % R != 0 -> per-tap kernel
    (3, 16, 128, 32, 32, 3, 1, 1),    # ragged: 3 images, 2 row groups each
]


SPLIT_CASES = [c for i, c in enumerate(CASES) if i % 3 == 1 or c[7] == 2]


@pytest.mark.parametrize("B,H,W,Cin,Cout,k,stride,mode", CASES)
def test_conv_parity(h, B, H, W, Cin, Cout, k, stride, mode):
    _run(h, B, H, W, Cin, Cout, k, stride, mode, False)


@pytest.mark.parametrize("B,H,W,Cin,Cout,k,stride,mode", SPLIT_CASES)
def test_conv_parity_split(h, B, H, W, Cin, Cout, k, stride, mode):
    """x2 precision: fp32 inputs stored as hi + lo fp16; the result must be fp32-grade:
    |err| <= 2^-20 |ref| + 1e-5 (two fp16 roundings of a residual, fp32 accumulation)."""
    _run(h, B, H, W, Cin, Cout, k, stride, mode, True)


@pytest.mark.parametrize("B,H,W,Cin,Cout,k,stride,mode", [c for c in CASES if c[3] % 32 == 0] +
                         [(1, 128, 128, 32, 32, 3, 1, 3), (1, 64, 64, 32, 64, 3, 1, 1), (1, 32, 32, 96, 96, 3, 1, 0)])
def test_conv_parity_f8(h, B, H, W, Cin, Cout, k, stride, mode):
    """f8 precision (R9): fp32 inputs stored as fp16 hi + e4m3 lo (x 2^6), the lo
    term multiplied by e5m2(W 2^-6) into the same fp32 accumulator. The reference applies
    exactly those roundings (torch's RNE float8 casts) to x, r and the lo weights, so what
    remains is the fp32 accumulation order and the f8 rounding of the stored output:
    |err| <= 2^-18 sum|terms| + 2^-14 |ref| + 2^-15. Dropping the lo term or mis-scaling it
    errs by ~2^-12 |ref| and fails."""
    _run(h, B, H, W, Cin, Cout, k, stride, mode, "f8")


def _f8_store(a):
    """fp32 -> stored f8 pair value: fp16 hi + e4m3 RNE-saturated lo (x 2^6) / 2^6."""
    import torch
    a32 = np.asarray(a, np.float32)
    hi = a32.astype(np.float16).astype(np.float32)
    lo = torch.from_numpy(((a32 - hi) * 64.0).astype(np.float32)).clamp(-448, 448)
    lo = lo.to(torch.float8_e4m3fn).to(torch.float64).numpy() / 64.0
    return hi.astype(np.float64) + lo, hi.astype(np.float64), lo


def _e5m2_lo_weights(w):
    import torch
    t = torch.from_numpy((np.asarray(w, np.float64) / 64.0).astype(np.float32))
    return t.to(torch.float8_e5m2).to(torch.float64).numpy() * 64.0


RC_CASES = [
    (1, 128, 128, 32, 32, 3, 1, 1),   # nz, row-chunked residual + output
    (2, 128, 128, 64, 64, 3, 1, 0),
    (1, 256, 256, 32, 64, 3, 2, 0),   # stride-2 over a row-chunked input (conv3s2_rc_kernel), RC output
    (2, 256, 256, 64, 128, 3, 2, 0),  # the level-1 down conv shape (BN = 128, R = 2)
    (1, 256, 128, 32, 32, 3, 2, 0),   # ragged-ish: 2 column blocks, BN = 32
    (1, 64, 64, 64, 32, 1, 1, 2),     # up-add, row-chunked output and skip
    (1, 128, 128, 128, 64, 1, 1, 2),  # the level-1 up-conv shape (two 32-channel epilogue chunks)
    (1, 128, 128, 32, 32, 1, 1, 0),   # 1x1 per-tap (the stem), row-chunked output
]


@pytest.mark.parametrize("split", [False, "x2", "f8"])
@pytest.mark.parametrize("B,H,W,Cin,Cout,k,stride,mode", RC_CASES)
def test_conv_parity_row_chunked(h, B, H, W, Cin, Cout, k, stride, mode, split):
    """Row-chunked residual / output layout ([B][H][16-B chunk][W][16 B]): the same
    values as NHWC, for every storage kind."""
    _run(h, B, H, W, Cin, Cout, k, stride, mode, split, rc=True)


@pytest.mark.parametrize("split", [False, "x2", "f8"])
@pytest.mark.parametrize("B,H,W,Cin,Cout,k,stride,mode", [(1, 128, 128, 128, 64, 1, 1, 2), (1, 128, 128, 64, 32, 1, 1, 2),
                                                          (1, 128, 128, 64, 64, 3, 1, 1)])
def test_conv_parity_rc_out_nhwc_res(h, B, H, W, Cin, Cout, k, stride, mode, split):
    """Row-chunked output with an NHWC residual / skip (the up-conv of a level whose skip is
    NHWC, the b-conv writing E_l)."""
    _run(h, B, H, W, Cin, Cout, k, stride, mode, split, rc=True, res_nhwc=True)


def _run(h, B, H, W, Cin, Cout, k, stride, mode, split, rc=False, res_nhwc=False):
    rng = np.random.default_rng(B * 1000 + H + Cin + Cout + k + stride + mode)
    x = rng.standard_normal((B, H, W, Cin)) if split else _f16(rng.standard_normal((B, H, W, Cin)))
    w = _f16(rng.standard_normal((Cout, k, k, Cin)) * np.sqrt(2.0 / (k * k * Cin)))
    b = rng.standard_normal(Cout).astype(np.float32).astype(np.float64) * 0.1
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    r = None
    if mode == 1:
        r = rng.standard_normal((B, Ho, Wo, Cout))
    elif mode == 2:
        r = rng.standard_normal((B, 2 * Ho, 2 * Wo, Cout))
    if r is not None and not split:
        r = _f16(r)
    if split:   # the GPU sees fp32-rounded inputs
        x = x.astype(np.float32).astype(np.float64)
        r = None if r is None else r.astype(np.float32).astype(np.float64)
    if split == "f8":
        _, xhi, xlo = _f8_store(x)
        rs = None if r is None else _f8_store(r)[0]
        wlo = _e5m2_lo_weights(w)
        pre = np.stack([nn.conv2d(xhi[i], w, b, stride) + nn.conv2d(xlo[i], wlo, np.zeros_like(b), stride)
                        for i in range(B)])
        if mode == 0:
            ref = np.maximum(pre, 0)
        elif mode == 1:
            ref = np.maximum(pre + rs, 0)
        elif mode == 2:
            ref = rs + np.stack([nn.up2(p) for p in pre])
        else:
            ref = pre if rs is None else pre + rs
        got = h.conv(x, w, b, stride=stride, r=r, mode=mode, split=split, rc=rc, res_nhwc=res_nhwc)
        ref_abs = _ref(np.abs(x), np.abs(w), np.abs(b), stride, None if r is None else np.abs(r),
                       3 if mode != 2 else 2)
        bound = 2.0 ** -18 * np.abs(ref_abs) + 2.0 ** -14 * np.abs(ref) + 2.0 ** -15
        err = np.abs(got - ref)
        assert got.shape == ref.shape
        assert (err <= bound).all(), f"max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
        return
    ref = _ref(x, w, b, stride, r, mode)
    got = h.conv(x, w, b, stride=stride, r=r, mode=mode, split=split, rc=rc, res_nhwc=res_nhwc)
    err = np.abs(got - ref)
    if split:
        # fp32 accumulation over K terms: |err| <= K eps32 sum|terms| (worst case); use the
        # sum of |terms| (conv of |x| with |w|) as the scale, plus the two output roundings
        ref_abs = _ref(np.abs(x), np.abs(w), np.abs(b), stride, None if r is None else np.abs(r),
                       3 if mode != 2 else 2)
        bound = 2.0 ** -18 * np.abs(ref_abs) + 2.0 ** -21 * np.abs(ref) + 1e-6
    else:
        bound = TOL_REL * np.abs(ref) + 1e-3
    assert got.shape == ref.shape
    assert (err <= bound).all(), f"max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
