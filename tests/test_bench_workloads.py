"""Host logic of bench.py's workload presets (SURVEY §8(f) N1 / N4 geometries)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_default_workload_is_one_call_over_all_tasks():
    w, groups = _bench().resolve_workload("cfg4")
    assert w.name == "cfg4_needle_biopsy"
    assert groups == [(256, list(range(6)))]


def test_paper_geometry_strides_per_scale():
    """40x windows at stride 256, 10x and 5x at stride 64; every task in exactly one call."""
    w, groups = _bench().resolve_workload("cfg4_paper")
    assert w.arch["fusion"] == "vote" and w.patch == 512
    by_stride = {S: sorted(w.scales[i] for i in idx) for S, idx in groups}
    assert by_stride == {256: [40], 64: [5, 5, 10, 10, 10]}
    assert sorted(i for _, idx in groups for i in idx) == list(range(len(w.scales)))
    # interior coverage (P/S)^2 = 64 windows fits the vote canvas' 16-bit count field
    assert (w.patch // 64) ** 2 < 1 << 16
    # each call's tasks are a contiguous run of the task list (one area slice per call)
    for _, idx in groups:
        assert idx == list(range(idx[0], idx[-1] + 1))


def test_oracle_pipeline_geometry_n4():
    w, groups = _bench().resolve_workload("cfg4_n4")
    assert (w.patch, w.stride, w.pad) == (256, 128, 2048)
    assert w.arch["fusion"] == "vote" and len(groups) == 1


def test_foreground_sweep_names():
    b = _bench()
    for f in (5, 25, 60, 95):
        w, groups = b.resolve_workload(f"cfg5_fg{f}")
        assert w.name == f"cfg5_sweep_fg{f}" and (w.H, w.W) == (40000, 40000)
        assert groups == [(256, list(range(6)))]


def test_stride_sweep_and_24_task_variant():
    """BASELINE configs[4] strides 512 / 384 / 256 and the cfg4 '6 classes at 4 scales' variant."""
    b = _bench()
    for S in (384, 512):
        w, groups = b.resolve_workload(f"cfg5_fg95_s{S}")
        assert w.stride == S and w.name == f"cfg5_sweep_fg95_s{S}" and groups == [(S, list(range(6)))]
    w, groups = b.resolve_workload("cfg4_24")
    assert len(w.scales) == 24 and sorted(zip(w.scales, w.classes)) == sorted(
        (s, c) for s in (5, 10, 20, 40) for c in range(6))
    assert [sorted(set(w.scales[i] for i in idx)) for _, idx in groups] == [[5], [10], [20], [40]]


def test_path_roofline_closed_form():
    """bench.path_roofline on a hand-made step: one call, 2 windows at f = 1 with one task."""
    import numpy as np
    b = _bench()
    from omniseg_inputs import workload
    w = workload(2)
    w.scales, w.classes = (10,), (2,)
    ids = [np.array([0, 1], np.uint32)]       # log2 f = 0 for both
    gsl = [(256, [10], [2], 0, 0, [0])]
    prof = {"flops": 2 * 98.3e9, "ms": 1.0, "launches": 1}
    pk = {"hbm_gbs": 6000.0, "bf16_tflops": 1600.0, "bf16_tflops_sustained": 1400.0}
    r = b.path_roofline(w, gsl, ids, prof, 1, 2, 1000.0, pk, "measured")
    P, H, W = 512, 4096, 4096
    F = 2 * (98.3e9 + P * P * (2 * 32 * 8 + 272))
    B = 3 * H * W + 2 * (3 + 8) * P * P + 9 * H * W
    assert abs(r["F_alg_tflop"] - F / 1e12) < 1e-9 and abs(r["B_alg_gb"] - B / 1e9) < 1e-9
    assert abs(r["T_roof_ms_sustained"] - max(F / 1.4e15, B / 6e12) * 1e3) < 1e-9
    assert r["bound"] == "tensor"
