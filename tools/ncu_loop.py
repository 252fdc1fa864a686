"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
instructions whose execution count equals COUNT (one loop body), with their
warp-stall samples and top stall reasons."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
count = int(sys.argv[2]) if len(sys.argv) > 2 else None
hdr = rows[1]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
names = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
if count is None:
    c = collections.Counter()
    for r in data:
        c[int(r[idx['Instructions Executed']] or 0)] += int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    for ex, s in sorted(c.items(), key=lambda x: -x[1])[:20]: print(ex, s)
    sys.exit()
tot = 0; agg = collections.Counter()
for r in data:
    ex = int(r[idx['Instructions Executed']] or 0)
    if ex != count: continue
    s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    tot += s
    br = {n: int(r[idx[n]] or 0) for n in names}
    agg.update(br)
    top = [f"{k[6:]}={v}" for k, v in sorted(br.items(), key=lambda x: -x[1])[:3] if v > 0]
    print(r[0][-5:], f"{s:5d}", r[1][:80], " ".join(top))
print("total samples", tot, dict(agg.most_common(8)))
