"""Kept-tile counts of the BASELINE configs computed by the ORACLE front end (used only
to extrapolate the oracle's timing sample in bench.py's reference / cpu_baseline legs).
Writes tests/golden/kept_tiles.json.   python scripts/oracle_tile_counts.py [cfg ...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from omniseg_inputs import arch_string, geometry, render, workload  # noqa: E402
from oracle import frontend as fe  # noqa: E402
from oracle import net as nn  # noqa: E402
from oracle import pipeline as op  # noqa: E402

out_path = os.path.join(ROOT, "tests", "golden", "kept_tiles.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {
    "_source": "kept-tile counts from the oracle front end (scripts/oracle_tile_counts.py)"}
for cfg in [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]:
    w = workload(cfg)
    g = geometry(w.slide)
    slide = np.concatenate([render(g, r, min(w.H, r + 4096)).numpy() for r in range(0, w.H, 4096)])
    tf = op.task_factors(nn.parse_arch(arch_string(w.arch)), w.scales)
    fr = op.front_end(slide, w.pad, w.patch, w.stride, [f for f, _ in tf])
    res[w.name] = len(fr["kept"])
    res[w.name + "_per_scale"] = {str(k): v for k, v in fr["grids"].items()}
    print(w.name, len(fr["kept"]), fr["grids"], flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
