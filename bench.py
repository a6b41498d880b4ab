"""Benchmark: slide-wise Omni-Seg prediction on B200 (BASELINE.json metric
"slide megapixels/sec (all classes) at 1/2/4/8 B200; sec per synthetic biopsy WSI").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--dtype fp16f8]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the oracle arm (CPU, bounded sample)

One step = one full pass of the hot path (upload excluded for `value`: the slide is
resident in HBM; pyramid, detection, tile selection, gather, trunk, GAP/controller,
head, stitch, finalize) over the whole synthetic slide; at N > 1 every rank segments
its row band (strong scaling: the WSI is fixed). `e2e` repeats the step through the
same C-ABI call with host buffers (H2D of the slide and D2H of prob/mask/area inside
the timed region). Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "slide megapixels/sec (all classes)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4",
                    help="cfg1..cfg5 (BASELINE.json configs; cfg5_fg5/25/60/95[_s384|_s512]: the foreground / "
                         "stride sweep; cfg4_24: 6 classes x 4 scales), "
                         "or a SURVEY §8(f) geometry on cfg4's slide: "
                         "cfg4_paper (N1: vote fusion, 40x S=256, 10x/5x S=64), "
                         "cfg4_n4 (N4: Oracle-pipeline geometry, 256 windows, S=128, pad 2048, vote)")
    ap.add_argument("--dtype", default=None,
                    help="fp16f8 (default: fp16 + e4m3 residual, parity-gated), fp16x2 (gated), fp16, bf16")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--arch", action="append", default=[], metavar="KEY=VALUE",
                    help="extra arch key (repeatable), e.g. --arch grp=1 --arch glev=2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="1 warmup + 1 step, for ncu")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# SURVEY §8(f) workloads on cfg4's slide. `groups`: (stride, magnifications) per
# omniseg_segment_slide call -- the API takes one stride per call, so the paper's per-scale
# strides (40x 256, 10x/5x 64) are two calls per step.
PRESETS = {
    # vthr: the paper's literal vote-count thresholds per scale code 5/10/20/40 ("set to 4" at
    # 10x/5x, "set to 1" at 40x; 20x has none -> majority), against the 2-D coverage, min(thr, cov)
    "cfg4_paper": dict(base=4, fusion="vote", vthr=(4, 4, 0, 1), groups=((256, (40,)), (64, (10, 5)))),
    "cfg4_n4": dict(base=4, fusion="vote", patch=256, stride=128, pad=2048),
}


def resolve_workload(name):
    """-> (Workload, [(stride, [task indices])]) for a --workload name."""
    from omniseg_inputs import workload
    pr = PRESETS.get(name)
    if pr is None and name.startswith("cfg5_fg"):
        # BASELINE configs[4] sweep point: cfg5_fg5/25/60/95, optionally _s384 / _s512 (stride sweep)
        parts = name[7:].split("_s")
        w = workload(5, fg_fraction=int(parts[0]) / 100)
        if len(parts) > 1:
            w.stride = int(parts[1])
            w.name += f"_s{w.stride}"
        return w, [(w.stride, list(range(len(w.scales))))]
    if name == "cfg4_24":
        # SURVEY §8(d) cfg4 variant "all 6 classes at 4 scales" (BASELINE configs[3]): 24 tasks, every
        # class at 5x / 10x / 20x / 40x; one call per scale (6 tasks each) so every call's fused head
        # runs only the tasks of its windows' scale
        from omniseg_inputs.arch import SCALE_CODES_4
        w = workload(4)
        w.name = "cfg4_24tasks"
        w.scales = tuple(s for s in SCALE_CODES_4 for _ in range(6))
        w.classes = tuple(c for _ in SCALE_CODES_4 for c in range(6))
        return w, [(w.stride, list(range(6 * k, 6 * k + 6))) for k in range(4)]
    if pr is None:
        w = workload(int(name.replace("cfg", "")))
        return w, [(w.stride, list(range(len(w.scales))))]
    w = workload(pr["base"])
    w.name = name
    w.arch["fusion"] = pr["fusion"]
    if "vthr" in pr:
        w.arch["vthr"] = pr["vthr"]
    for k in ("patch", "stride", "pad"):
        if k in pr:
            setattr(w, k, pr[k])
    if "groups" not in pr:
        return w, [(w.stride, list(range(len(w.scales))))]
    groups = [(S, [i for i, s in enumerate(w.scales) if s in mags]) for S, mags in pr["groups"]]
    assert sorted(i for _, g in groups for i in g) == list(range(len(w.scales)))
    return w, groups


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ reference arm (oracle)
def oracle_sample(w, slide_rows_fn, n_tiles=1, strip=512):
    """Oracle (as it stands) on a bounded sample of the workload: the front end on a
    `strip`-row window and `n_tiles` windows through trunk + head + stitch; the whole-slide
    time is extrapolated linearly by rows (front end) and by the kept-tile count."""
    from oracle import frontend as fe
    from oracle import net as onn
    from oracle import pipeline as op
    from omniseg_inputs import arch_string
    arch = onn.parse_arch(arch_string(w.arch))
    net = onn.unpack_weights(arch, w.weights())
    tf = op.task_factors(arch, w.scales)
    H, W = w.H, w.W
    win = slide_rows_fn(0, min(H, strip))
    t0 = time.perf_counter()
    fr = op.front_end(win, w.pad, w.patch, w.stride, [f for f, _ in tf])
    t_fe = time.perf_counter() - t0
    lv = fe.level(fr["padded"], 1)
    tasks = [(c, s) for c, (f, s) in zip(w.classes, tf) if f == 1] or [(w.classes[0], tf[0][1])]
    t1 = time.perf_counter()
    acc = np.zeros((w.patch, w.patch))
    cnt = np.zeros((w.patch, w.patch), np.int64)
    for i in range(n_tiles):
        oy = 0
        ox = min(i * w.stride, lv.shape[1] - w.patch)
        p = onn.predict_tile(net, arch, lv[oy:oy + w.patch, ox:ox + w.patch], tasks)
        for k in range(p.shape[0]):
            op.stitch_add(acc, cnt, p[k], 0, 0)
    t_tile = (time.perf_counter() - t1) / n_tiles
    return t_fe, t_tile


def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from omniseg_inputs import geometry, render
    if a.workload in PRESETS or a.workload == "cfg4_24":
        print(json.dumps({"impl": "reference", "unavailable": f"{a.workload}: the oracle arm is timed on cfg1..cfg5"}))
        return 0
    w, _ = resolve_workload(a.workload)
    g = geometry(w.slide)
    rows = lambda r0, r1: render(g, r0, r1).numpy()  # noqa: E731
    n_kept = tile_estimate(w)
    times = []
    cores = len(os.sched_getaffinity(0))
    for i in range(a.warmup + a.steps):
        t_fe, t_tile = oracle_sample(w, rows)
        T = t_fe * w.H / 512 + t_tile * n_kept
        if i >= a.warmup:
            times.append(T)
    T = statistics.median(times)
    v = w.H * w.W / 1e6 / T
    out = {"metric": METRIC, "value": v, "unit": "Mpx/s", "impl": "reference", "n_gpus": 0, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": T * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": w.name, "H": w.H, "W": w.W, "patch": w.patch, "stride": w.stride,
                      "pad": w.pad, "tasks": len(w.scales), "kept_tiles_used": n_kept},
           "cpu_baseline": {"value": v, "unit": "Mpx/s", "cores": cores, "kind": "oracle",
                            "sample": f"per step: oracle front end on a 512-row strip + 1 kept-size 512^2 "
                                      f"window through trunk+head+stitch (fp64 numpy), extrapolated by rows "
                                      f"and by {n_kept} kept tiles"},
           "e2e": {"value": v, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def tile_estimate(w):
    """Kept-tile count of the workload as computed by the ORACLE front end
    (tests/golden/kept_tiles.json, written by scripts/oracle_tile_counts.py); only used to
    extrapolate the oracle's timing sample. Falls back to the SURVEY §8(d) estimate."""
    est = {"cfg5_sweep_fg95": 31874}
    p = os.path.join(ROOT, "tests", "golden", "kept_tiles.json")
    try:
        with open(p) as f:
            return json.load(f)[w.name]
    except (OSError, KeyError, ValueError):
        return est.get(w.name, 1000)


# ------------------------------------------------------------------ our arm
def path_roofline(w, gsl, kept_ids, prof, steps, rank_windows, ms, pk, pk_kind):
    """north_star's whole-path roofline: T_roof = max(F_alg / tensor peak,
    B_alg / HBM bandwidth) over the algorithmic work of the step, and T_roof / T_step.
      F_alg = sum over kept windows of the trunk's convolution FLOPs (2 M N K with the real channel
              counts, from the live per-conv profile: per window = profiled FLOPs / windows run)
              + the dynamic head (precls 2 C0 8 + 2 * 136 per task of the window's scale, per px);
      B_alg = 3 H W (slide read) + 4 (Hp/f)(Wp/f) per level f > 1 written + 3 P^2 per kept window
              (window read) + 8 P^2 per window-task (canvas read-modify-write) + 9 Ht Wt per task
              (finalize: canvas read, prob + mask write)."""
    H, W, P, pad = w.H, w.W, w.patch, w.pad
    Hp, Wp = (H + 2 * pad + 127) // 128 * 128, (W + 2 * pad + 127) // 128 * 128
    mag = w.arch["slide_mag"]
    C0 = w.arch["base"]
    per_window = prof["flops"] / max(steps * rank_windows, 1)
    F = B = 0.0
    for (S, sc, cl, n0, n1, idx), ids in zip(gsl, kept_ids):
        lf = (np.asarray(ids, np.uint32) >> 30).astype(np.int64)
        facs = sorted(set(mag // s for s in sc))
        B += 3.0 * H * W + sum(4.0 * (Hp // f) * (Wp // f) for f in facs if f > 1)
        for f in facs:
            nk = int((lf == f.bit_length() - 1).sum())
            ntask = sum(1 for s in sc if mag // s == f)
            F += nk * (per_window + P * P * (2.0 * C0 * 8 + ntask * 272.0))
            B += nk * (3.0 * P * P + ntask * 8.0 * P * P)
        for s in sc:
            f = mag // s
            B += 9.0 * ((H + f - 1) // f) * ((W + f - 1) // f)
    bw = pk.get("hbm_gbs", 6556.5) * 1e9
    out = {"F_alg_tflop": F / 1e12, "B_alg_gb": B / 1e9, "T_step_ms": ms,
           "bound": "tensor" if F / (pk.get("bf16_tflops_sustained", 1376.7) * 1e12) > B / bw else "hbm",
           "peak_kind": pk_kind}
    for kind, key in (("sustained", "bf16_tflops_sustained"), ("burst", "bf16_tflops")):
        tf = pk.get(key)
        if tf:
            t_roof = max(F / (tf * 1e12), B / bw) * 1e3
            out[f"T_roof_ms_{kind}"] = t_roof
            out[f"frac_{kind}"] = t_roof / ms if ms else None
    return out


# committed ncu launch-list summaries of the cfg4 command, newest first
NCU_SUMMARIES = ("r02z_cfg4_ncu_summary.json", "r02_cfg4_ncu_summary.json")


def hbm_kernels():
    """Per-kernel DRAM throughput of the HBM-bound kernels from the committed ncu capture of the
    cfg4 command (the newest profiles/r02*_cfg4_ncu_summary.json, scripts/summarize_ncu_r02.py)."""
    for name in NCU_SUMMARIES:
        p = os.path.join(ROOT, "profiles", name)
        try:
            with open(p) as f:
                return json.load(f).get("hbm_kernels")
        except (OSError, ValueError):
            continue
    return None


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from omniseg_inputs import arch_string, geometry, render
    from paper_2305_14566_b200 import Omniseg
    from paper_2305_14566_b200 import dist as D
    from paper_2305_14566_b200 import lib as L

    w, groups = resolve_workload(a.workload)
    if world > 1 and len(groups) > 1:
        raise SystemExit(f"{a.workload}: per-scale strides run at N=1 only (bands follow one stride)")
    if a.dtype:
        w.arch["dtype"] = a.dtype
    if a.batch:
        w.arch["batch"] = a.batch
    for kv in a.arch:
        k, v = kv.split("=", 1)
        w.arch[k] = int(v) if v.lstrip("-").isdigit() else v
    H, W = w.H, w.W
    Hp = (H + 2 * w.pad + 127) // 128 * 128
    fmax = max(w.arch["slide_mag"] // s for s in w.scales)
    cuts = D.band_cuts(Hp, world, w.stride)
    if world > 1:
        row0, row1 = cuts[rank], cuts[rank + 1]
        b0, b1 = D.band_slide_rows(H, w.pad, w.patch, fmax, row0, row1)
    else:
        row0, row1, b0, b1 = 0, Hp, 0, H
    dev = torch.device("cuda", local)
    t0 = time.time()
    g = geometry(w.slide)
    slide = render(g, b0, b1, device=dev, chunk_rows=2048) if b1 > b0 else torch.zeros((1, W, 3), torch.uint8,
                                                                                         device=dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    h = Omniseg(arch_string(w.arch), w.weights())
    stream = torch.cuda.current_stream(dev)
    h.set_stream(stream.cuda_stream)
    # outputs (owned canvas rows of every task), laid out group by group
    ncan, gsl = 0, []
    for S, idx in groups:
        n0 = ncan
        for i in idx:
            f = w.arch["slide_mag"] // w.scales[i]
            r0t, r1t = L.band_rows(H, row0, row1, w.pad, f)
            ncan += (r1t - r0t) * ((W + f - 1) // f)
        gsl.append((S, [w.scales[i] for i in idx], [w.classes[i] for i in idx], n0, ncan, idx))
    prob = torch.empty(max(ncan, 1), dtype=torch.float32, device=dev)
    mask = torch.empty(max(ncan, 1), dtype=torch.uint8, device=dev)
    # N > 1, device-resident: the bands are gathered into full-slide outputs on rank 0 (NCCL)
    nfull = sum(((H + f - 1) // f) * ((W + f - 1) // f) for f in (w.arch["slide_mag"] // s for s in w.scales))
    full_prob = torch.empty(nfull if (world > 1 and rank == 0) else 1, dtype=torch.float32, device=dev)
    full_mask = torch.empty(nfull if (world > 1 and rank == 0) else 1, dtype=torch.uint8, device=dev)
    area = torch.zeros(len(w.scales), dtype=torch.int64, device=dev)
    D.init_comm(h, world, rank)

    def step(src, p_out, m_out, a_out, gather=True, record=None):
        """One step; record: list receiving each call's kept-window ids (untimed warm-up only)."""
        if world > 1:
            h.segment_band(src, H, W, row0, row1, w.pad, w.patch, w.stride, w.scales, w.classes, p_out, m_out, a_out)
            if record is not None:
                record.append(h.tiles())
            if gather:   # device-resident outputs: the band gather to rank 0 (host outputs stay per rank)
                h.gather_bands(0, H, W, w.pad, cuts, w.scales, p_out, m_out, full_prob, full_mask)
            return
        for S, sc, cl, n0, n1, idx in gsl:
            if len(gsl) == 1:
                h.segment_slide(src, H, W, w.pad, w.patch, S, sc, cl, p_out, m_out, a_out)
            else:
                h.segment_slide(src, H, W, w.pad, w.patch, S, sc, cl, p_out[n0:n1], m_out[n0:n1],
                                a_out[idx[0]:idx[-1] + 1])
            if record is not None:
                record.append(h.tiles())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    nwarm = max(1, a.warmup if not a.profile_only else 1)
    kept_ids = []
    for i in range(nwarm):
        step(slide, prob, mask, area, record=kept_ids if i == nwarm - 1 else None)
    rank_windows = sum(len(k) for k in kept_ids)
    if world > 1:   # whole-job unique windows: the union of the ranks' (overlapping) window sets
        allk = [None] * world
        dist.all_gather_object(allk, [k.tolist() for k in kept_ids])
        kept_ids = [np.array(sorted(set(v for r in allk for k in r for v in k)), np.uint32)]
    n_tiles = sum(len(k) for k in kept_ids)
    steps = 1 if a.profile_only else a.steps
    clocks = Clocks(local)
    h.set_profile(True)
    barrier()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step(slide, prob, mask, area)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / steps
    prof = h.profile()
    h.set_profile(False)
    launches = int(h.timings()[10])
    t_ms = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms = float(t_ms.item())
    value = H * W / 1e6 / (ms / 1e3)

    # ---- end to end: host pinned input, host outputs, copies inside the timed region
    e2e = None
    if not a.no_e2e and not a.profile_only:
        hslide = torch.empty(slide.shape, dtype=torch.uint8, pin_memory=True)
        hslide.copy_(slide)
        hprob = torch.empty(prob.shape, dtype=torch.float32, pin_memory=True)
        hmask = torch.empty(mask.shape, dtype=torch.uint8, pin_memory=True)
        harea = torch.zeros(area.shape, dtype=torch.int64, pin_memory=True)
        step(hslide, hprob, hmask, harea, gather=False)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step(hslide, hprob, hmask, harea, gather=False)
        e1.record(stream)
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        ems = float(ems.item())
        e2e = {"value": H * W / 1e6 / (ems / 1e3), "unit": "Mpx/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(hslide.numel()), "d2h_bytes_per_step": int(ncan * 5 + 8 * len(w.scales)),
               "note": "host pinned slide in, host prob/mask/area out, through omniseg_segment_slide/band"}

    pk, pk_kind = peaks()
    achieved = prof["flops"] / (prof["ms"] / 1e3) / 1e12 if prof["ms"] > 0 else 0.0
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    # DRAM traffic per conv launch from the committed ncu capture of the same launch shapes
    # (batch-64 launches of the cfg2 profile run: dram__bytes_read.sum + dram__bytes_write.sum)
    traffic, traffic_src = None, None
    for tname in NCU_SUMMARIES + ("r01o_cfg2_summary.json",):
        tpath = os.path.join(ROOT, "profiles", tname)
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            traffic = tj.get("conv_dram_bytes_per_launch")
            traffic_src = "profiles/%s (ncu, %d conv launches)" % (tname, tj.get("conv_launches", 0))
            break
    roof = {"bound": "tensor", "kernel": "tcgen05 conv family (stem_tc / conv3_nz / conv3s2_rc / conv_tc kernels)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
            "peak_kind": f"{pk_kind} bf16 sustained (fp16 kind::f16 nominal ratio 1.0)",
            "traffic": traffic, "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic_src,
            "conv_share_of_step": (prof["ms"] / steps) / ms if ms else None,
            "alg_flops_per_launch": prof["flops"] / max(prof["launches"], 1),
            "avg_launch_ms": prof["ms"] / max(prof["launches"], 1)}
    roof["path"] = path_roofline(w, gsl, kept_ids, prof, steps, rank_windows, ms, pk, pk_kind)
    hk = hbm_kernels()
    if hk:
        roof["hbm_kernels"] = hk
    cpu = None
    if a.workload in PRESETS or a.workload == "cfg4_24":
        cpu = {"value": None, "unit": "Mpx/s", "cores": 0, "kind": "oracle",
               "sample": "not run: the oracle baseline is timed on cfg1..cfg5 (bench.py --workload cfg4)"}
    elif rank == 0 and world == 1 and not a.no_cpu and not a.profile_only:
        try:
            strip, nt = 1024, 2  # ~10 s of CPU work
            t_fe, t_tile = oracle_sample(w, lambda r0, r1: render(g, r0, r1).numpy(), n_tiles=nt, strip=strip)
            n_or = tile_estimate(w)
            T = t_fe * H / strip + t_tile * n_or
            cpu = {"value": H * W / 1e6 / T, "unit": "Mpx/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                   "sample": f"oracle (fp64 numpy) front end on a {strip}-row strip ({t_fe:.2f} s) + {nt} 512^2 "
                             f"windows through trunk+head+stitch ({t_tile:.2f} s each), extrapolated to {H} rows "
                             f"and {n_or} kept tiles (oracle tile plan)"}
        except Exception as e:  # the baseline must never break the bench line
            cpu = {"value": None, "unit": "Mpx/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                   "sample": f"failed: {e}"}
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "Mpx/s", "n_gpus": world, "steps": steps,
               "warmup": a.warmup, "ms_per_step": ms, "sec_per_wsi": ms / 1e3, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": w.arch["dtype"], "data": "synthetic",
               "config": {"workload": w.name, "H": H, "W": W, "patch": w.patch,
                          "stride": w.stride if len(gsl) == 1 else {"x".join(map(str, g[1])): g[0] for g in gsl},
                          "pad": w.pad, "fusion": w.arch.get("fusion", "mean"),
                          "tasks": len(w.scales), "kept_tiles": n_tiles, "batch": w.arch["batch"],
                          "schedule": (f"L2-resident groups of {w.arch['grp']} windows for levels < "
                                       f"{w.arch.get('glev', 2)}" if w.arch.get("grp") else "batch-wide"),
                          "parallelism": (f"row-bands x{world} + NCCL band gather to rank 0" if world > 1
                                          else "single GPU"),
                          "l2": "inputs larger than L2 (slide %.1f GB, canvases %.1f GB)"
                                % (slide.numel() / 1e9, ncan * 5 / 1e9),
                          "slide_gen_s": round(gen_s, 1)},
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches * steps,
               "clocks": clk, "stage_ms": [round(x, 3) for x in h.timings()[:9].tolist()]}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
