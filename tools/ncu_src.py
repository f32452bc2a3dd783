"""Print the SASS source page of an ncu report (csv) with stall samples per
instruction: python tools/ncu_src.py report.csv [min_samples]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
mins = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = {}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = r[ix["Instructions Executed"]]
    top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    for v, h in top:
        tot[h] = tot.get(h, 0) + v
    if s >= mins:
        print(f"{r[ix['Address']]:>6} {s:6d} {ex:>9} {r[ix['Source']][:60]:60s} "
              + " ".join(f"{h}={v}" for v, h in top if v))
print("totals:", sorted(((v, k) for k, v in tot.items()), reverse=True)[:10])
