"""Summarise an `ncu --page source --csv` export: stall reasons per instruction-execution-count class
(one class ~ one warp role of a warp-specialised kernel) and the top stalled instructions."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
cls = collections.defaultdict(lambda: collections.Counter())
ninst = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    e = int(r[ix["Instructions Executed"]] or 0)
    ninst[e] += 1
    for h in reasons:
        cls[e][h] += int(r[ix[h]] or 0)
top = sorted(cls, key=lambda e: -sum(cls[e].values()))[: int(sys.argv[2]) if len(sys.argv) > 2 else 8]
for e in top:
    c = cls[e]
    tot = sum(c.values())
    print(f"exec={e:10d} ninstr={ninst[e]:4d} samples={tot:7d} " +
          " ".join(f"{k[6:]}={v}" for k, v in c.most_common(6)))
