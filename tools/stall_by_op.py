"""Aggregate ncu source-page (SASS) stall samples by opcode and stall reason.

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > src.csv
    python tools/stall_by_op.py src.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in data:
    if len(r) < len(hdr):
        continue
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    for h in reasons:
        try:
            v = int(r[hdr.index(h)] or 0)
        except ValueError:
            continue
        agg[o][h[6:]] += v
        tot[h[6:]] += v
allv = sum(tot.values())
print("total samples", allv, {k: round(v / allv, 3) for k, v in tot.most_common(8)})
for o, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"{o:10s} {s / allv:6.3f}", {k: round(v / allv, 3) for k, v in c.most_common(4)})
