"""Summarise an ncu `--page source --csv --print-source sass` export: warp-stall samples and
executed instructions grouped by SASS opcode, and the hottest instructions.

    python tools/sass_profile.py gpurun_out/ncu2/cfg3_svd_rr.source.csv [top]
"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    out = []
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        out.append(dict(zip(hdr, r)))
    return hdr, out


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr, rows = load(path)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_op = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
    tot = 0.0
    for r in rows:
        src = r["Source"].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        s = num(r["Warp Stall Sampling (All Samples)"])
        by_op[op][0] += s
        by_op[op][1] += num(r["Instructions Executed"])
        for c in stall_cols:
            by_op[op][2][c] += num(r[c])
        tot += s
    print(f"total samples {tot:.0f}")
    print(f"{'op':10s} {'samples%':>8s} {'inst(M)':>9s}  top stalls")
    for op, (s, n, st) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:top]:
        tops = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{op:10s} {100 * s / tot:8.2f} {n / 1e6:9.3f}  " + ", ".join(f"{k[6:]} {100 * v / tot:.1f}" for k, v in tops))
    print("\nhottest instructions:")
    for r in sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]:
        s = num(r["Warp Stall Sampling (All Samples)"])
        st = sorted(((c, num(r[c])) for c in stall_cols), key=lambda kv: -kv[1])[:2]
        print(f"{100 * s / tot:6.2f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} " +
              ", ".join(f"{k[6:]} {v:.0f}" for k, v in st))


if __name__ == "__main__":
    main()
