"""Pins for the oracle stitch/finalize (O10-O11) and end-to-end closed forms."""
import numpy as np

from oracle import frontend as fe
from oracle import net as nn
from oracle import pipeline as op
from omniseg_inputs import arch_dict, arch_string, blank_slide, make_slide, make_weights, param_count, workload


def _coverage_1d(E, P, S, pad, n):
    """Per-axis coverage of canvas index i by tiles with origins(E, P, S), shifted by pad."""
    cov = np.zeros(n, np.int64)
    for o in fe.origins(E, P, S):
        lo, hi = max(0, o - pad), min(n, o - pad + P)
        cov[lo:hi] += 1
    return cov


def test_uniform_p_gives_uniform_canvas_and_product_counts():
    """north_star closed form: uniform tile probabilities give a uniform canvas and the
    overlap weights (1/cnt) sum to exactly 1; with every tile kept the count canvas is
    the outer product of the per-axis coverage counts."""
    H, W, P, S, pad = 300, 420, 64, 32, 40
    Hp, Wp = fe.padded_extent(H, W, pad)
    s, c = np.zeros((H, W)), np.zeros((H, W), np.int64)
    tiles = [(oy, ox) for oy in fe.origins(Hp, P, S) for ox in fe.origins(Wp, P, S)]
    for oy, ox in tiles:
        op.stitch_add(s, c, np.full((P, P), 0.375), oy - pad, ox - pad)
    prob, mask = op.finalize(s, c)
    assert (c == np.outer(_coverage_1d(Hp, P, S, pad, H), _coverage_1d(Wp, P, S, pad, W))).all()
    assert (prob == 0.375).all() and mask.sum() == 0
    # weights 1/cnt per covering tile sum to exactly 1 where covered
    wsum = np.zeros((H, W))
    for oy, ox in tiles:
        op.stitch_add(wsum, np.zeros((H, W), np.int64), np.ones((P, P)), oy - pad, ox - pad)
    assert (wsum == c).all()


def test_stitch_order_independent_and_dropped_tiles():
    rng = np.random.default_rng(0)
    H, W, P = 100, 90, 32
    tiles = [(int(rng.integers(-20, 90)), int(rng.integers(-20, 80))) for _ in range(40)]
    ps = [rng.integers(0, 2 ** 10, (P, P)) / 2 ** 10 for _ in tiles]   # dyadic: exact sums
    s1, c1 = np.zeros((H, W)), np.zeros((H, W), np.int64)
    for (y, x), p in zip(tiles, ps):
        op.stitch_add(s1, c1, p, y, x)
    s2, c2 = np.zeros((H, W)), np.zeros((H, W), np.int64)
    for i in rng.permutation(len(tiles)):
        op.stitch_add(s2, c2, ps[i], *tiles[i])
    assert (s1 == s2).all() and (c1 == c2).all()
    prob, _ = op.finalize(s1, c1)
    assert (prob[c1 == 0] == 0).all()


def test_blank_slide_empty_masks():
    """north_star invariant: an all-background slide yields empty masks."""
    w = workload(1)
    s = blank_slide(512, 512).numpy()
    r = op.segment_slide(s, w.weights(), arch_string(w.arch), 64, 256, 128, (1,), (0,))
    assert r["kept"] == [] and r["area"] == [0] and (r["prob"][0] == 0).all()


def test_constant_network_end_to_end():
    """Zero conv weights and zero controller weights, bias-only head: theta = bc, F = b_pre,
    so every kept tile predicts the same p = sigmoid(z0) (closed form), the canvas equals
    p exactly where a kept tile covers it and 0 elsewhere."""
    a = arch_dict(levels=3, base=8, ncls=1, scale_codes=(1,), slide_mag=1)
    blob = np.zeros(param_count(a))
    arch = nn.parse_arch(arch_string(a))
    net = nn.unpack_weights(arch, blob)
    # fill in the bias slots via a view of the same blob
    theta = np.concatenate([np.eye(8).ravel(), np.zeros(8), np.eye(8).ravel(), np.zeros(8),
                            np.full(8, 0.25), [-1.0]])
    net["ctrl"][1][:] = theta
    net["precls"][1][:] = np.linspace(-1, 2, 8)
    z0 = 0.25 * np.maximum(np.linspace(-1, 2, 8), 0).sum() - 1.0
    p0 = 1.0 / (1.0 + np.exp(-z0))
    s = make_slide(workload(1).slide).numpy()[:512, :512]
    r = op.segment_slide(s, blob, arch_string(a), 64, 128, 64, (1,), (0,))
    prob = r["prob"][0]
    cov = r["cnt"][0] > 0
    assert len(r["kept"]) > 0
    np.testing.assert_allclose(prob[cov], p0, rtol=1e-14)
    assert (prob[~cov] == 0).all()
    assert r["area"][0] == (int(cov.sum()) if p0 >= 0.5 else 0)


def test_covering_tiles_matches_count_canvas():
    w = workload(1)
    s = make_slide(w.slide).numpy()
    fr = op.front_end(s, w.pad, w.patch, w.stride, [1])
    H, W = s.shape[:2]
    sums, cnt = np.zeros((H, W)), np.zeros((H, W), np.int64)
    for (f, oy, ox) in fr["kept"]:
        op.stitch_add(sums, cnt, np.zeros((w.patch, w.patch)), oy - w.pad, ox - w.pad)
    rng = np.random.default_rng(1)
    for _ in range(50):
        y, x = int(rng.integers(0, H)), int(rng.integers(0, W))
        assert len(op.covering_tiles(fr["kept"], 1, w.pad, w.patch, y, x)) == cnt[y, x]


# ---------------------------------------------------------------- hard-vote fusion
def test_vote_of_threshold_is_at_least_half():
    """the paper's thresholds (1 of 2, 4 of 8) are 'at least half' -- a window votes
    positive iff p >= 1/2, ties included."""
    p = np.array([0.0, 0.4999999, 0.5, 0.5000001, 1.0])
    assert op.vote_of(p).tolist() == [0, 0, 1, 1, 1]


def test_vote_fusion_matches_brute_force_majority():
    """Vote fraction and mask against an explicit per-pixel count of covering windows and
    positive votes (brute force over tiles), including exact ties (2 of 4 -> positive)."""
    rng = np.random.default_rng(5)
    H, W, P = 40, 44, 16
    tiles = [(int(rng.integers(-8, 36)), int(rng.integers(-8, 40))) for _ in range(30)]
    ps = [rng.random((P, P)) for _ in tiles]
    s, c = np.zeros((H, W)), np.zeros((H, W), np.int64)
    for (y, x), p in zip(tiles, ps):
        op.stitch_add(s, c, op.vote_of(p), y, x)
    prob, mask = op.finalize(s, c)
    for yy in range(H):
        for xx in range(W):
            votes = cov = 0
            for (y, x), p in zip(tiles, ps):
                if y <= yy < y + P and x <= xx < x + P:
                    cov += 1
                    votes += int(p[yy - y, xx - x] >= 0.5)
            assert c[yy, xx] == cov
            assert prob[yy, xx] == (votes / cov if cov else 0.0)
            assert mask[yy, xx] == int(cov > 0 and 2 * votes >= cov)


def test_vote_equals_thresholded_mean_where_one_window_covers():
    """End to end (cfg1): where exactly one kept window covers a pixel, the vote fraction is
    that window's decision, i.e. the mean-fusion probability thresholded at 1/2."""
    w = workload(1)
    slide = make_slide(w.slide).numpy()
    a = arch_string(w.arch)
    rm = op.segment_slide(slide, w.weights(), a, w.pad, w.patch, w.stride, w.scales, w.classes)
    rv = op.segment_slide(slide, w.weights(), a, w.pad, w.patch, w.stride, w.scales, w.classes, fusion="vote")
    one = rm["cnt"][0] == 1
    assert one.sum() > 1000
    assert (rv["prob"][0][one] == (rm["prob"][0][one] >= 0.5)).all()
    k = rv["prob"][0] * rm["cnt"][0]  # vote fractions are (integer votes) / cnt
    assert np.allclose(k, np.round(k), atol=1e-9)


# ---------------------------------------------------------------- literal vote-count threshold (arch vthr)
def _vote_sim(tiles, ps, H, W, P, thr):
    """Brute force: explicit per-pixel counters over every tile (S:311 'brute-force simulator')."""
    votes = np.zeros((H, W), np.int64)
    cov = np.zeros((H, W), np.int64)
    for (y, x), p in zip(tiles, ps):
        for yy in range(max(0, y), min(H, y + P)):
            for xx in range(max(0, x), min(W, x + P)):
                cov[yy, xx] += 1
                votes[yy, xx] += int(p[yy - y, xx - x] >= 0.5)
    mask = np.zeros((H, W), np.uint8)
    for yy in range(H):
        for xx in range(W):
            c = cov[yy, xx]
            mask[yy, xx] = int(c > 0 and votes[yy, xx] >= min(thr, c))
    return votes, cov, mask


def test_vote_count_threshold_brute_force_and_monotone():
    """P:97 literal thresholds ('set to 1' at 40x, 'set to 4' at 10x/5x) applied to the 2-D
    coverage with the clamp min(thr, coverage): against the per-pixel brute force
    on random windows; raising the threshold never turns a 0 pixel into a 1."""
    rng = np.random.default_rng(11)
    H, W, P = 36, 40, 12
    tiles = [(int(rng.integers(-6, 32)), int(rng.integers(-6, 36))) for _ in range(40)]
    ps = [rng.random((P, P)) for _ in tiles]
    s, c = np.zeros((H, W)), np.zeros((H, W), np.int64)
    for (y, x), p in zip(tiles, ps):
        op.stitch_add(s, c, op.vote_of(p), y, x)
    prev = None
    for thr in (1, 2, 4, 8, 64):
        votes, cov, mask = _vote_sim(tiles, ps, H, W, P, thr)
        prob, m = op.finalize_vote_count(s, c, thr)
        assert (c == cov).all() and (s == votes).all()
        assert (m == mask).all(), thr
        assert (prob == np.where(cov > 0, votes / np.maximum(cov, 1), 0)).all()
        if prev is not None:
            assert not (m & ~prev).any()
        prev = m.astype(bool)


def test_vote_count_threshold_spec_40x_example():
    """40x configuration (extent 4096, window 512, stride 256 -> 225 tiles, threshold 1),
    predictor positive only in tiles whose origin x = 0: a pixel covered by such a tile gets
    >= 1 vote -> 1; pixels covered only by other tiles -> 0."""
    E, P, S = 4096, 512, 256
    org = fe.origins(E, P, S)
    assert len(org) ** 2 == 225
    s, c = np.zeros((E, E)), np.zeros((E, E), np.int64)
    for oy in org:
        for ox in org:
            op.stitch_add(s, c, np.full((P, P), 1.0 if ox == 0 else 0.0), oy, ox)
    _, m = op.finalize_vote_count(s, c, 1)
    exp = np.zeros((E, E), np.uint8)
    exp[:, :P] = 1
    assert (m == exp).all()
    assert (c[P:E - P, P:E - P] == 4).all()       # interior 2-D coverage (window / stride)^2


def test_vote_count_threshold_end_to_end_per_scale():
    """segment_slide with vthr: each task uses its scale code's threshold; thr = 1 makes a
    pixel positive iff any covering window votes positive."""
    w = workload(1)
    slide = make_slide(w.slide).numpy()
    w.arch["fusion"] = "vote"
    rm = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes)
    w.arch["vthr"] = (1,)
    r1 = op.segment_slide(slide, w.weights(), arch_string(w.arch), w.pad, w.patch, w.stride, w.scales, w.classes)
    assert (r1["prob"][0] == rm["prob"][0]).all()
    assert (r1["mask"][0] == (rm["prob"][0] > 0)).all()
    assert r1["mask"][0].sum() >= rm["mask"][0].sum()
