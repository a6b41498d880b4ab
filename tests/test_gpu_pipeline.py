"""GPU end-to-end parity through the C ABI against the oracle (north_star gates):
tile lists and foreground masks bit-exact; per-pixel |p_gpu - p_oracle| <= 1e-2;
masks agree on >= 99.9% of pixels and every disagreement sits where the oracle
probability is within 1e-2 of 0.5."""
import numpy as np
import pytest

from omniseg_inputs import arch_string, blank_slide, make_slide, random_tiles, workload
from oracle import frontend as fe
from oracle import net as nn
from oracle import pipeline as op

pytestmark = pytest.mark.gpu

P_TOL = 1e-2


def unpack_tiles(ids, Hp, Wp, P, S):
    out = []
    for v in ids.tolist():
        lf, ty, tx = v >> 30, (v >> 15) & 0x7FFF, v & 0x7FFF
        f = 1 << lf
        out.append((f, min(ty * S, Hp // f - P), min(tx * S, Wp // f - P)))
    return out


def check_prob_mask(p_gpu, m_gpu, p_ref, m_ref, tag=""):
    d = np.abs(p_gpu.astype(np.float64) - p_ref)
    assert d.max() <= P_TOL, f"{tag} max |dp| = {d.max():.4g}"
    dis = m_gpu != m_ref
    agree = 1.0 - dis.mean()
    assert agree >= 0.999, f"{tag} mask agreement {agree:.5f}"
    if dis.any():
        assert (np.abs(p_ref[dis] - 0.5) <= P_TOL).all(), f"{tag} mask flip away from 0.5"
    return d.max(), agree


def run_gpu(w, slide):
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(w.arch), w.weights())
    H, W = slide.shape[:2]
    n = sum(h.output_size(H, W, s) for s in w.scales)
    prob = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    area = np.zeros(len(w.scales), np.uint64)
    h.segment_slide(slide, H, W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, area)
    return h, prob, mask, area


def split(arr, H, W, w, arch):
    out, o = [], 0
    for s in w.scales:
        f = arch["slide_mag"] // s
        n = ((H + f - 1) // f) * ((W + f - 1) // f)
        out.append(arr[o:o + n].reshape((H + f - 1) // f, (W + f - 1) // f))
        o += n
    return out


_REF = {}


def _cfg1_ref():
    if "cfg1" not in _REF:
        w = workload(1)
        slide = make_slide(w.slide).numpy()
        _REF["cfg1"] = (slide, op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride,
                                                w.scales, w.classes))
    return _REF["cfg1"]


@pytest.fixture(scope="module")
def cfg1(gpu_lib):
    """The x2 precision mode (fp16x2: fp32-grade activations, R9), gated; the default
    fp16f8 is gated by test_cfg1_f8_gated and the full-size tests."""
    w = workload(1)
    w.arch["dtype"] = "fp16x2"
    slide, ref = _cfg1_ref()
    h, prob, mask, area = run_gpu(w, slide)
    return w, slide, ref, h, prob, mask, area


def test_cfg1_f8_gated(gpu_lib):
    """fp16f8 precision (fp16 hi + e4m3 lo activations, R9): the full gates --
    tile list / fg bit-exact, |dp| <= 1e-2, masks >= 99.9% with flips only near 0.5."""
    w = workload(1)
    w.arch["dtype"] = "fp16f8"
    slide, ref = _cfg1_ref()
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    Hp, Wp = fe.padded_extent(H, W, w.pad)
    assert unpack_tiles(h.tiles(), Hp, Wp, w.patch, w.stride) == ref["kept"]
    dmax, agree = check_prob_mask(prob.reshape(H, W), mask.reshape(H, W), ref["prob"][0], ref["mask"][0], "f8")
    print(f"fp16f8: max |dp| {dmax:.4g}, mask agreement {agree:.5f}")


def check_votes(ref, p_gpu, m_gpu, pad, P, task=0, f=1, tag=""):
    """Vote fusion gate: the GPU vote fraction may differ from the oracle's only by votes of
    windows whose oracle p is within 1e-2 of 1/2 (a decision fp16f8 rounding may flip): at
    every pixel, |votes_gpu - votes_ref| <= #(covering windows with |p - 1/2| <= 1e-2); a mask
    may differ only where such a window exists. Returns (fraction-equal share, mask agreement)."""
    cnt = ref["cnt"][task]
    p_ref = ref["prob"][task]
    dv = np.rint(np.abs(p_gpu.astype(np.float64) - p_ref) * cnt).astype(np.int64)
    bad = (dv > 0) | (m_gpu != ref["mask"][task])
    ys, xs = np.nonzero(bad)
    for cy, cx in zip(ys.tolist(), xs.tolist()):
        near = 0
        for k in op.covering_tiles(ref["kept"], f, pad, P, cy, cx):
            pk = ref["windows"][k][task][cy + pad // f - k[1], cx + pad // f - k[2]]
            near += abs(pk - 0.5) <= 1e-2
        assert near >= max(1, dv[cy, cx]), (tag, cy, cx, int(dv[cy, cx]), near)
    same = (np.abs(p_gpu.astype(np.float64) - p_ref) <= 1e-6).mean()
    agree = (m_gpu == ref["mask"][task]).mean()
    return same, agree


def test_cfg1_tensor_core_head_gated(gpu_lib):
    """The optional tcgen05 dynamic head (arch headtc=1: precls folded into layer 1, W1' D0 as
    fp16 hi/lo MMAs) under the same gates as the default head."""
    w = workload(1)
    w.arch["headtc"] = 1
    slide, ref = _cfg1_ref()
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    dmax, agree = check_prob_mask(prob.reshape(H, W), mask.reshape(H, W), ref["prob"][0], ref["mask"][0], "headtc")
    print(f"headtc: max |dp| {dmax:.4g}, mask agreement {agree:.5f}")


def test_cfg1_vote_fusion(gpu_lib):
    """Hard majority-vote fusion (arch fusion=vote) against the oracle's vote mode:
    every window votes p >= 1/2; the canvas holds the vote fraction, the mask is 'at least
    half'. Every difference must be explained by windows whose oracle p is within 1e-2 of 1/2
    (check_votes), and fractions / masks agree on >= 99.9 % of pixels."""
    w = workload(1)
    w.arch["fusion"] = "vote"
    slide, _ = _cfg1_ref()
    ref = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes,
                           keep_windows=True)
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    same, agree = check_votes(ref, prob.reshape(H, W), mask.reshape(H, W), w.pad, w.patch, tag="vote")
    print(f"vote: fraction-equal {same:.5f}, mask agreement {agree:.5f}")
    assert same >= 0.999 and agree >= 0.999
    assert int(area[0]) == int(mask.sum())


def test_cfg1_vote_count_threshold(gpu_lib):
    """The paper's literal vote-count threshold (arch vthr; P:97 'set to 1' at 40x): mask =
    votes >= min(thr, coverage), against the oracle's finalize_vote_count, near-1/2 rule."""
    w = workload(1)
    w.arch["fusion"] = "vote"
    w.arch["vthr"] = (1,)
    slide, _ = _cfg1_ref()
    ref = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes,
                           keep_windows=True)
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    same, agree = check_votes(ref, prob.reshape(H, W), mask.reshape(H, W), w.pad, w.patch, tag="vthr")
    m = mask.reshape(H, W)
    assert (m == (prob.reshape(H, W) > 0)).all()       # thr 1: any positive vote
    assert same >= 0.999 and agree >= 0.999
    assert int(area[0]) == int(m.sum())


def _vote_case(**geom):
    w = workload(1)
    w.arch["fusion"] = "vote"
    for k, v in geom.items():
        setattr(w, k, v)
    slide, _ = _cfg1_ref()
    ref = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes,
                           keep_windows=True)
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    Hp, Wp = fe.padded_extent(H, W, w.pad)
    assert unpack_tiles(h.tiles(), Hp, Wp, w.patch, w.stride) == ref["kept"]
    same, agree = check_votes(ref, prob.reshape(H, W), mask.reshape(H, W), w.pad, w.patch, tag=str(geom))
    assert same >= 0.999 and agree >= 0.999, (same, agree)
    assert int(area[0]) == int(mask.sum())
    return ref, same, agree


def test_cfg1_vote_dense_stride64(gpu_lib):
    """SURVEY N1's dense geometry (S = 64 at 10x/5x, 'at least half' of the covering
    windows): stride P/4, so an interior pixel is covered by up to 16 kept windows -- beyond the
    mean mode's 15-window count field, inside the vote mode's 16-bit one."""
    ref, same, agree = _vote_case(stride=64)
    assert ref["cnt"][0].max() == 16
    print(f"vote S=64: {len(ref['kept'])} tiles, fraction-equal {same:.5f}, mask agreement {agree:.5f}")


def test_cfg1_oracle_pipeline_geometry_n4(gpu_lib):
    """SURVEY N4 (the original pipeline's 2048-px padding and 256^2 windows),
    half-window stride and majority vote: tile plan bit-exact, votes as above."""
    ref, same, agree = _vote_case(pad=2048, patch=256, stride=128)
    print(f"N4 geometry: {len(ref['kept'])} tiles, fraction-equal {same:.5f}, mask agreement {agree:.5f}")


def test_cfg1_component_removal_and_fg_mask(gpu_lib):
    """SURVEY N2 (arch fgmin / maskfg): the level-8 foreground loses its components below
    fgmin pixels (GPU union-find vs the oracle's labelling, bit-exact), the window plan follows
    (bit-exact), and the output masks are ANDed with the foreground."""
    w = workload(1)
    w.arch["fgmin"] = 700      # cfg1's foreground components: 621, 741, 2043 level-8 px
    w.arch["maskfg"] = 1
    slide, _ = _cfg1_ref()
    ref = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes)
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    Hp, Wp = fe.padded_extent(H, W, w.pad)
    fg, t, gpad = h.fgmask()
    assert t == ref["t"] and (fg == ref["fg"]).all()
    assert int(ref["fg"].sum()) == 741 + 2043
    assert unpack_tiles(h.tiles(), Hp, Wp, w.patch, w.stride) == ref["kept"]
    check_prob_mask(prob.reshape(H, W), mask.reshape(H, W), ref["prob"][0], ref["mask"][0], "fgmin")
    assert int(area[0]) == int(mask.sum())


def test_overlay_render_bit_exact(gpu_lib):
    """SURVEY N3 (omniseg_render_overlay): the 40x overlay and the 10x downsample of the masks a
    segment call produced, bit-exact against oracle/render.py on the same masks -- including
    several tasks of different scales and classes overlapping (precedence) and a ragged 10x edge."""
    from oracle import render as rd
    w = workload(1)
    slide, _ = _cfg1_ref()
    slide = slide[:1021, :1018].copy()           # ragged: neither side a multiple of 4
    H, W = slide.shape[:2]
    a = dict(w.arch, ncls=6, scale_codes=(5, 10, 40), slide_mag=40)
    from omniseg_inputs import make_weights
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(a), make_weights(a, 1))
    scales, classes = (40, 10, 5, 40), (2, 0, 5, 4)
    sizes = [h.output_size(H, W, s) for s in scales]
    mask = np.zeros(sum(sizes), np.uint8)
    h.segment_slide(slide, H, W, 64, 128, 64, scales, classes, None, mask, None)
    rng = np.random.default_rng(0)
    mask |= (rng.random(mask.shape) < 0.05).astype(np.uint8)   # more overlap between classes
    out40 = np.zeros((H, W, 3), np.uint8)
    out10 = np.zeros(((H + 3) // 4, (W + 3) // 4, 3), np.uint8)
    h.render_overlay(slide, H, W, mask, scales, classes, out40, out10)
    factors = [40 // s for s in scales]
    ms, o = [], 0
    for n, f in zip(sizes, factors):
        ms.append(mask[o:o + n].reshape((H + f - 1) // f, (W + f - 1) // f))
        o += n
    ref40 = rd.overlay_40x(slide, rd.merge_40x(ms, factors, H, W), classes)
    assert (out40 == ref40).all()
    assert (out10 == rd.downsample_4(ref40)).all()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_cfg1_16bit_storage_numerics_report(gpu_lib, dtype):
    """Plain 16-bit activation storage (BASELINE configs' 'bf16 activations', and fp16):
    NOT gated at 1e-2 -- the random network amplifies storage rounding beyond it
    (R9, reproduced bit-for-bit by scripts/emulate_storage.py). Reported, with
    tile lists still bit-exact and a sanity bound on |dp|."""
    w = workload(1)
    w.arch["dtype"] = dtype
    slide, ref = _cfg1_ref()
    h, prob, mask, area = run_gpu(w, slide)
    H, W = slide.shape[:2]
    Hp, Wp = fe.padded_extent(H, W, w.pad)
    assert unpack_tiles(h.tiles(), Hp, Wp, w.patch, w.stride) == ref["kept"]
    d = np.abs(prob.reshape(H, W).astype(np.float64) - ref["prob"][0])
    agree = (mask.reshape(H, W) == ref["mask"][0]).mean()
    print(f"{dtype}: max |dp| {d.max():.4g}, p99.99 {np.quantile(d, 0.9999):.4g}, mask agreement {agree:.5f}")
    assert d.max() <= (0.06 if dtype == "fp16" else 0.3)


def test_cfg1_tiles_and_fg_bit_exact(cfg1):
    w, slide, ref, h, prob, mask, area = cfg1
    H, W = slide.shape[:2]
    Hp, Wp = fe.padded_extent(H, W, w.pad)
    assert unpack_tiles(h.tiles(), Hp, Wp, w.patch, w.stride) == ref["kept"]
    fg, t, gpad = h.fgmask()
    assert t == ref["t"] and gpad == ref["g_pad"]
    assert (fg == ref["fg"]).all()


def test_cfg1_prob_mask_area(cfg1):
    w, slide, ref, h, prob, mask, area = cfg1
    H, W = slide.shape[:2]
    P = split(prob, H, W, w, w.arch)
    M = split(mask, H, W, w, w.arch)
    for t in range(len(w.scales)):
        check_prob_mask(P[t], M[t], ref["prob"][t], ref["mask"][t], f"task{t}")
        assert int(area[t]) == int(M[t].sum())
        assert abs(int(area[t]) - ref["area"][t]) <= 0.001 * P[t].size


def test_blank_slide_empty(gpu_lib):
    w = workload(1)
    s = blank_slide(512, 512).numpy()
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(w.arch), w.weights())
    prob = np.ones(512 * 512, np.float32)
    mask = np.ones(512 * 512, np.uint8)
    area = np.ones(1, np.uint64)
    h.segment_slide(s, 512, 512, 64, 256, 128, (1,), (0,), prob, mask, area)
    assert len(h.tiles()) == 0 and area[0] == 0 and not prob.any() and not mask.any()


def test_predict_tiles_tiny_net(gpu_lib):
    """Trunk + head on given windows (no stitch) vs the oracle: F, g and p."""
    from paper_2305_14566_b200 import Omniseg
    w = workload(1)
    arch = nn.parse_arch(arch_string(w.arch))
    net = nn.unpack_weights(arch, w.weights())
    tiles = random_tiles(3, 256, 11).numpy()
    h = Omniseg(arch_string(w.arch), w.weights())
    p, F, g = h.predict_tiles(tiles, [(0, 0)], with_F=True, with_g=True, c_bottleneck=32)
    for i in range(3):
        Fr, Er = nn.trunk(net, arch, tiles[i])
        gr = nn.gap(Er)
        pr = nn.head(Fr, nn.controller(net, arch, gr, 0, 0))
        scale = np.abs(Fr).max()
        eF = np.abs(F[i] - Fr).max() / scale
        eg = np.abs(g[i] - gr).max() / np.abs(gr).max()
        ep = np.abs(p[i, 0] - pr).max()
        print(f"window {i}: F rel {eF:.3g}, g rel {eg:.3g}, max |dp| {ep:.3g}")
        assert eF <= 2 ** -10, eF
        assert eg <= 2 ** -10, eg
        assert ep <= 1e-2, ep


@pytest.mark.slow
def test_predict_tiles_cfg2_net(gpu_lib):
    """One 512x512 window through the config-2 network (the bench network)."""
    from paper_2305_14566_b200 import Omniseg
    w = workload(2)
    arch = nn.parse_arch(arch_string(w.arch))
    net = nn.unpack_weights(arch, w.weights())
    tiles = random_tiles(1, 512, 12).numpy()
    h = Omniseg(arch_string(w.arch), w.weights())
    tasks = [(2, 1), (3, 1), (5, 1)]
    p, F, g = h.predict_tiles(tiles, tasks, with_F=True, with_g=True, c_bottleneck=512)
    Fr, Er = nn.trunk(net, arch, tiles[0])
    gr = nn.gap(Er)
    eF = np.abs(F[0] - Fr).max() / np.abs(Fr).max()
    eg = np.abs(g[0] - gr).max() / np.abs(gr).max()
    print(f"F rel {eF:.3g}, g rel {eg:.3g}")
    assert eF <= 2 ** -10, eF
    assert eg <= 2 ** -10, eg
    for k, (c, s) in enumerate(tasks):
        pr = nn.head(Fr, nn.controller(net, arch, gr, c, s))
        d = np.abs(p[0, k] - pr)
        print(f"task {k}: max |dp| {d.max():.4g}  p99.99 {np.quantile(d, 0.9999):.4g}")
        assert d.max() <= 1e-2


def test_invalid_calls_fail_cleanly_and_the_handle_recovers(gpu_lib):
    """Boundary error behaviour (include/omniseg.h): every invalid call returns a nonzero code
    with a message and leaves the handle usable -- the next valid call gives the same result
    as a fresh handle."""
    from paper_2305_14566_b200 import Omniseg, lib
    w = workload(1)
    slide, _ = _cfg1_ref()
    H, W = slide.shape[:2]
    h = Omniseg(arch_string(w.arch), w.weights())
    n = h.output_size(H, W, w.scales[0])
    prob = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    bad = [
        (dict(patch=250), "multiple"),              # patch not a multiple of 16 / 8
        (dict(stride=0), "stride"),                 # stride out of range
        (dict(stride=w.patch * 2), "stride"),       # stride > patch
        (dict(pad=3), "pad"),                       # pad not a multiple of 8
        (dict(scales=(7,)), "scale"),               # scale not in scale_codes
        (dict(classes=(99,)), "class"),             # class index out of range
        (dict(H=1), "H and W"),                     # degenerate slide
    ]
    for over, msg in bad:
        a = dict(H=H, W=W, pad=w.pad, patch=w.patch, stride=w.stride, scales=w.scales, classes=w.classes)
        a.update(over)
        with pytest.raises(lib.OmnisegError, match=msg):
            h.segment_slide(slide, a["H"], a["W"], a["pad"], a["patch"], a["stride"], a["scales"], a["classes"],
                            prob, mask, None)
    with pytest.raises(lib.OmnisegError):
        h.segment_slide(None, H, W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, None)
    h.segment_slide(slide, H, W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, None)
    _, p2, m2, _ = run_gpu(w, slide)
    assert (prob == p2).all() and (mask == m2).all()


def _shift_identity_net(levels, base, bc=None, dtype="fp16f8"):
    from special_nets import shift_identity_net
    return shift_identity_net(levels, base, bc=bc, dtype=dtype)


@pytest.mark.parametrize("levels, base, P, dtype", [(3, 8, 256, "fp16f8"), (5, 32, 512, "fp16f8"),
                                                   (5, 32, 512, "fp16x2")])
def test_shift_identity_network_bit_exact(gpu_lib, levels, base, P, dtype):
    """The single-tap identity network of tests/test_oracle_net.py, generalised to L levels
    (stem tap (0, 1): y = x shifted down one row; enc0 = RB with conv_a = I, conv_b = I/2, so
    E0 = 1.5 y; down0 tap (1, 2), deeper downs centre taps; identity up-convs and precls):
        F[i, j, c] = 1.5 (y[i, j] + sum_{l=1}^{L-1} y[2^l (i >> l), 2^l (j >> l) + 1]),  c < 3,
    through the CUDA trunk (the bench network's kernels at levels=5, base=32, P=512): every
    value is exact in the fp16 + e4m3 storage and in fp32 accumulation, so F must match
    BIT-EXACTLY -- this pins the kernels' spatial layout (tap orientation, padding, the
    stride-2 sample, up x2, skips) independently of rounding. theta = 0 (zero controller)
    gives p = sigmoid(0) = 1/2 exactly."""
    from paper_2305_14566_b200 import Omniseg
    a, net, blob = _shift_identity_net(levels, base, dtype=dtype)
    arch = nn.parse_arch(arch_string(a))
    tiles = random_tiles(2, P, 21).numpy()
    h = Omniseg(arch_string(a), blob)
    p, F, _ = h.predict_tiles(tiles, [(0, 0)], with_F=True)
    i = np.arange(P)[:, None]
    j = np.arange(P)[None, :]
    for t in range(2):
        y = np.zeros((P, P, 3))
        y[1:] = tiles[t][:-1]
        exp = y.copy()
        for l in range(1, levels):
            exp += y[(i >> l) << l, ((j >> l) << l) + 1]
        exp *= 1.5
        if levels == 3:
            Fr, _ = nn.trunk(net, arch, tiles[t])
            assert (Fr[:, :, :3] == exp).all()  # the oracle meets the closed form
        assert (F[t, :, :, :3] == exp).all(), np.abs(F[t, :, :, :3] - exp).max()
        assert (F[t, :, :, 3:] == 0).all()
    assert (p == 0.5).all()


@pytest.mark.parametrize("levels, base, P, S, pad, headtc", [(3, 8, 256, 128, 128, 0), (5, 32, 512, 256, 256, 0),
                                                             (3, 8, 256, 128, 128, 1), (5, 32, 512, 256, 256, 1)])
def test_shift_identity_network_slide_parity(gpu_lib, levels, base, P, S, pad, headtc):
    """The identity network end to end through omniseg_segment_slide (fused gather + stem,
    trunk, fused head + stitch, finalize) on the cfg1 slide, with theta = bc chosen so that
    z = F_0 / 256 - 2 (W1 = W2 = I, W3 = e_0 / 256, b3 = -2): F is exact on both sides, so
    the stitched probabilities may differ only by the fp32 sigmoid and the 2^-20 fixed point
    -- |dp| <= 2e-6 instead of the 1e-2 gate for random networks -- and the masks agree
    except where the oracle's mean is within 2e-6 of 1/2. Pins the window gather, the
    stem's window-relative padding and the stitch geometry; (5, 32, 512) runs the bench
    network's kernels (32-channel fused stem, no-swizzle / stride-2 / per-tap convs, fused
    head + stitch)."""
    theta = np.zeros(153)
    theta[0:64] = np.eye(8).ravel()
    theta[72:136] = np.eye(8).ravel()
    theta[144] = 1.0 / 256
    theta[152] = -2.0
    a, net, blob = _shift_identity_net(levels, base, bc=theta)
    if headtc:
        a["headtc"] = 1   # the optional tcgen05 head (layer 1 + precls as MMAs): exact here too
    w = workload(1)
    slide, _ = _cfg1_ref()
    H, W = slide.shape[:2]
    ref = op.segment_slide(slide, blob, arch_string(a), pad, P, S, w.scales, w.classes)
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(a), blob)
    prob = np.zeros(H * W, np.float32)
    mask = np.zeros(H * W, np.uint8)
    h.segment_slide(slide, H, W, pad, P, S, w.scales, w.classes, prob, mask, None)
    p_ref = ref["prob"][0]
    d = np.abs(prob.reshape(H, W).astype(np.float64) - p_ref)
    assert d.max() <= 2e-6, d.max()
    covered = ref["cnt"][0] > 0
    pc = p_ref[covered]
    assert covered.mean() > 0.3 and pc.min() < 0.3 and pc.max() > 0.7 and pc.std() > 0.02  # informative
    dis = mask.reshape(H, W) != ref["mask"][0]
    assert (np.abs(p_ref[dis] - 0.5) <= 2e-6).all()


def test_shift_identity_network_vote_exact(gpu_lib):
    """Vote fusion with the identity network and z = F_0 / 256 - 2: z is exact in
    fp32 on the GPU (F exact, a power-of-two scale), so every window's vote equals the
    oracle's and the vote fractions and masks must agree EXACTLY, dense stride included
    (S = 64: up to 16 covering windows)."""
    theta = np.zeros(153)
    theta[0:64] = np.eye(8).ravel()
    theta[72:136] = np.eye(8).ravel()
    theta[144] = 1.0 / 256
    theta[152] = -2.0
    a, net, blob = _shift_identity_net(3, 8, bc=theta)
    a["fusion"] = "vote"
    w = workload(1)
    slide, _ = _cfg1_ref()
    H, W = slide.shape[:2]
    ref = op.segment_slide(slide, blob, arch_string(a), w.pad, w.patch, 64, w.scales, w.classes)
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(a), blob)
    prob = np.zeros(H * W, np.float32)
    mask = np.zeros(H * W, np.uint8)
    area = np.zeros(1, np.uint64)
    h.segment_slide(slide, H, W, w.pad, w.patch, 64, w.scales, w.classes, prob, mask, area)
    assert ref["cnt"][0].max() == 16
    d = np.abs(prob.reshape(H, W).astype(np.float64) - ref["prob"][0])
    assert d.max() <= 1e-7, d.max()
    assert (mask.reshape(H, W) == ref["mask"][0]).all()
    assert int(area[0]) == int(ref["mask"][0].sum())
    assert 0.05 < ref["mask"][0].mean() < 0.95
