"""Summarise round-2 ncu launch lists of the cfg4 bench command into profiles/:
per kernel: launches, mean ms (ncu: serialised, cold), DRAM bytes per launch, achieved DRAM GB/s
and its fraction of the measured HBM copy peak (MEASURED_PEAKS.json hbm_gbs); the conv family's
DRAM bytes per launch (bench.py roofline.traffic) and the HBM-bound kernels' fractions
(bench.py roofline.hbm_kernels).

    python scripts/summarize_ncu_r02.py OUT_PREFIX launches1.csv [launches2.csv ...]"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TSCALE = {"usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "ns": 1e-6, "second": 1e3}
BSCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
HBM_BOUND = ("pyramid", "finalize", "stem_tc", "median7", "gap_kernel", "overlay")


def rows(path):
    h = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r and "Metric Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            yield dict(zip(h, r))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    out, paths = sys.argv[1], sys.argv[2:]
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        peak = 6556.5
    agg = collections.OrderedDict()
    for p in paths:
        per = collections.OrderedDict()
        for d in rows(p):
            m = per.setdefault((d["ID"], d["Kernel Name"]), {})
            v = num(d["Metric Value"])
            u = d["Metric Unit"]
            if d["Metric Name"] == "gpu__time_duration.sum":
                m["ms"] = v * TSCALE.get(u, 1.0)
            elif d["Metric Name"].startswith("dram__bytes"):
                m["bytes"] = m.get("bytes", 0.0) + v * BSCALE.get(u, 1.0)
        for (_, name), m in per.items():
            short = re.sub(r"^void |\(.*$", "", name).replace("osg::", "").replace("(anonymous namespace)::", "")
            a = agg.setdefault(short, [0, 0.0, 0.0])
            a[0] += 1
            a[1] += m.get("ms", 0.0)
            a[2] += m.get("bytes", 0.0)
    tab = ["| kernel | launches | mean ms | DRAM GB / launch | DRAM GB/s | % of HBM peak |", "|---|---|---|---|---|---|"]
    hbm = {}
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = b / (t / 1e3) / 1e9 if t > 0 else 0.0
        tab.append(f"| `{k}` | {c} | {t / c:.4f} | {b / c / 1e9:.4f} | {gbs:.0f} | {100 * gbs / peak:.1f}% |")
        if any(s in k for s in HBM_BOUND):
            key = next(s for s in HBM_BOUND if s in k)
            hbm[key] = {"dram_gbs": round(gbs, 1), "frac": round(gbs / peak, 4), "launches": c}
    conv = {k: v for k, v in agg.items() if "conv" in k or "stem_tc" in k}
    cl = sum(v[0] for v in conv.values())
    cb = sum(v[2] for v in conv.values())
    summ = {"conv_launches": cl, "conv_dram_bytes_per_launch": cb / cl if cl else None,
            "hbm_peak_gbs": peak, "hbm_kernels": hbm, "source": [os.path.basename(p) for p in paths]}
    with open(out + ".json", "w") as f:
        json.dump(summ, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write("# ncu launch list summary (" + ", ".join(os.path.basename(p) for p in paths) + ")\n\n")
        f.write("ncu serialises launches and runs them cold (`--clock-control none`): compare shares and bytes, "
                "not absolute step times.\n\n")
        f.write("\n".join(tab) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    sys.exit(main())
