"""Summarise the ncu captures of a round into profiles/ (launch list -> per-kernel shares and
DRAM bytes per launch; full capture -> per-kernel key metrics).
    python scripts/summarize_ncu.py <launches.csv> <full_raw.csv> <out_prefix>"""
import collections
import csv
import json
import sys


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


def launches(path):
    per = collections.OrderedDict()
    units = {}
    for d in rows(path):
        key = (d["ID"], d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = num(d["Metric Value"])
        units[d["Metric Name"]] = d["Metric Unit"]
    return per, units


def main():
    lpath, fpath, out = sys.argv[1:4]
    per, units = launches(lpath)
    scale = {"usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "ns": 1e-6}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0]
        t = m.get("gpu__time_duration.sum", 0) * scale.get(units.get("gpu__time_duration.sum"), 1)
        byt = (m.get("dram__bytes_read.sum", 0) * bscale.get(units.get("dram__bytes_read.sum"), 1) +
               m.get("dram__bytes_write.sum", 0) * bscale.get(units.get("dram__bytes_write.sum"), 1))
        a = agg[short]
        a[0] += 1
        a[1] += t
        a[2] += byt
    # namespace-qualified names, or (captures filtered with -k regex:osg::) every kernel listed
    ours = {k: v for k, v in agg.items() if "osg::" in k} or dict(agg)
    tot = sum(v[1] for v in ours.values())
    conv = {k: v for k, v in ours.items() if any(s in k for s in ("conv", "stem_tc"))}
    conv_launch = sum(v[0] for v in conv.values())
    conv_bytes = sum(v[2] for v in conv.values())
    lines = ["| kernel | launches | ms (ncu, serialised) | share | DRAM GB per launch |", "|---|---|---|---|---|"]
    for k, (c, t, b) in sorted(ours.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k.replace('void ', '')}` | {c} | {t:.2f} | {100 * t / tot:.1f}% | {b / c / 1e9:.3f} |")
    summary = {
        "conv_launches": conv_launch,
        "conv_dram_bytes_per_launch": conv_bytes / max(conv_launch, 1),
        "conv_share_of_kernel_time": sum(v[1] for v in conv.values()) / tot,
        "source": lpath,
    }
    # full capture
    full = []
    h, u = None, None
    for r in csv.reader(open(fpath)):
        if "Kernel Name" in r and h is None:
            h = r
            continue
        if h and u is None and len(r) == len(h) and r[0] == "":
            u = dict(zip(h, r))  # the units row
            continue
        if h and len(r) == len(h) and r[0] not in ("", "ID") and not r[0].startswith("("):
            d = dict(zip(h, r))
            if not d.get("Kernel Name"):
                continue
            g = lambda k: num(d.get(k, "nan"))  # noqa: E731
            gu = lambda k: g(k) * {**scale, **bscale}.get((u or {}).get(k, ""), 1.0)  # noqa: E731
            full.append((d["Kernel Name"].split("(")[0].replace("void ", ""), gu("gpu__time_duration.sum"),
                         gu("dram__bytes_read.sum") / 1e9, gu("dram__bytes_write.sum") / 1e9,
                         g("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                         g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                         g("lts__throughput.avg.pct_of_peak_sustained_elapsed")))
    flines = ["| kernel (one batch, launch order) | ms | DRAM read GB | DRAM write GB | tensor pipe active % | DRAM % | L2 % |",
              "|---|---|---|---|---|---|---|"]
    for f in full:
        flines.append("| `%s` | %.3f | %.3f | %.3f | %.1f | %.1f | %.1f |" % f)
    open(out + "_launches.md", "w").write("\n".join(lines) + "\n")
    open(out + "_full.md", "w").write("\n".join(flines) + "\n")
    json.dump(summary, open(out + "_summary.json", "w"), indent=1)
    print("\n".join(lines[:25]))
    print("\n".join(flines))
    print(summary)


if __name__ == "__main__":
    main()
