"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

python tools/launch_summary.py gpurun_out/launches_cfg3.csv [...]  -> markdown table on stdout
"""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def summarise(path):
    rows = load(path)
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        if "<" in r["Kernel Name"]:
            k = r["Kernel Name"][: r["Kernel Name"].find(">(") + 1] or k
        a = agg.setdefault(k, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
        a[1] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-3)
    tot = sum(v[1] for v in agg.values())
    out = [f"### {path}", "", "| launches | total us | share | avg us | grid | block | kernel |",
           "|---:|---:|---:|---:|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0]:.1f} | {v[2]} | {v[3]} | `{k}` |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
