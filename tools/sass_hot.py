"""Stall hot spots by SASS window: python tools/sass_hot.py source.csv [window] [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]; iS = hdr.index("Source"); iE = hdr.index("Instructions Executed"); iSm = hdr.index("# Samples")
cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
idx = {c: hdr.index(c) for c in cols}
body = [r for r in rows[2:] if len(r) > iE]
tot = sum(int(float(r[iSm])) for r in body)
agg = []
for i in range(0, len(body), win):
    seg = body[i:i + win]
    s = sum(int(float(r[iSm])) for r in seg)
    ex = max(int(float(r[iE])) for r in seg)
    st = {c: sum(int(float(r[idx[c]])) for r in seg) for c in cols}
    tp = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    agg.append((s, i, ex, tp, seg[0][iS].strip()[:40]))
for s, i, ex, tp, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% @{i:5d} exec {ex:9d} {src:40s}", ', '.join(f"{c[6:]} {v}" for c, v in tp))
if len(sys.argv) > 4:
    a, b = int(sys.argv[4]), int(sys.argv[5])
    for r in body[a:b]:
        print(r[iE], r[iSm], r[iS].strip()[:90])
