"""Opcode mix (warp-level instructions executed, stall samples) from an ncu source page CSV.
python tools/sass_mix.py gpurun_out/ncu/cfg3_svd_reg.source.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE, iSm = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
ex = collections.Counter(); sm = collections.Counter()
for r in rows[2:]:
    if len(r) <= iE: continue
    op = r[iS].strip().split()
    if not op: continue
    o = op[0]
    if o.startswith("@"): o = op[1]
    o = o.split(".")[0]
    try:
        ex[o] += int(float(r[iE])); sm[o] += int(float(r[iSm]))
    except ValueError:
        pass
T = sum(ex.values()); S = sum(sm.values())
print(f"total warp-inst {T:.3e}, samples {S}")
for o, v in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {v:14d} {100*v/T:5.1f}%  samples {100*sm[o]/S:5.1f}%")
