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
