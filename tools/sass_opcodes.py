"""Executed-instruction counts by SASS opcode class for each ncu capture (from the
`--page source --csv --print-source sass` exports): the evidence that the block kernels issue
FP64 tensor-core MMAs (DMMA) fed by cp.async (LDGSTS), and what the Jacobi / QR tiers issue.

    python tools/sass_opcodes.py gpurun_out/ncu2 > profiles/sass_opcodes_r02.md
"""
import csv
import os
import sys
from collections import Counter

CLASSES = ["DMMA", "HMMA", "DFMA", "DMUL", "DADD", "MUFU", "SHFL", "FSEL", "LDS", "STS", "LDG", "STG", "LDGSTS",
           "UBLKCP", "UTMALDG", "SYNCS", "BAR", "LDSM"]


def count(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ii = hdr.index("Instructions Executed")
    si = hdr.index("Source")
    c = Counter()
    kernel = rows[0][1] if len(rows[0]) > 1 else ""
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        src = r[si].strip()
        if not src:
            continue
        op = src.split()[0]
        if op.startswith("@"):
            op = src.split()[1]
        try:
            n = float(r[ii])
        except ValueError:
            continue
        c[op.split(".")[0]] += n
        c["_total"] += n
    return kernel, c


def main(src):
    print("| capture | kernel | warp-instr executed (M) | " + " | ".join(CLASSES) + " |")
    print("|---|---|---:|" + "---:|" * len(CLASSES))
    for f in sorted(os.listdir(src)):
        if not f.endswith(".source.csv"):
            continue
        kernel, c = count(os.path.join(src, f))
        k = kernel.split("(")[0].replace("void ", "")[:48]
        cells = " | ".join(f"{c[x] / 1e6:.2f}" if c[x] else "0" for x in CLASSES)
        print(f"| {f[:-11]} | `{k}` | {c['_total'] / 1e6:.1f} | {cells} |")
    print("\n(millions of warp-level instructions executed in the captured launch; DMMA = FP64 tensor-core "
          "mma.sync.m8n8k4, LDGSTS = cp.async global->shared, UBLKCP = cp.async.bulk (1-D TMA), UTMALDG = cp.async.bulk.tensor (2-D tensor-map TMA), SYNCS = mbarrier ops)")


if __name__ == "__main__":
    main(sys.argv[1])
