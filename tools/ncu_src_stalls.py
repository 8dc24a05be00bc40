"""Summarise an `ncu --page source --csv --print-source sass` export: for each kernel in it, stall reasons per
instruction-execution-count class (one class ~ one warp role of a warp-specialised kernel) and the top stalled
instructions.  Usage: ncu_src_stalls.py src.csv [classes] [top_instructions]"""
import collections
import csv
import sys


def sections(rows):
    cur = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "?", "rows": []}
            yield cur
        elif cur is not None:
            cur["rows"].append(r)


def summarise(name, rows, nclass, ntop):
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    if not reasons:   # newer ncu: stall columns are named after the reason without the stall_ prefix
        reasons = [h for h in hdr if h.startswith("Warp Stall Sampling (All Samples)") is False and "(All Samples)" in h]
    cls = collections.defaultdict(collections.Counter)
    ninst = collections.Counter()
    inst = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        try:
            e = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        ninst[e] += 1
        tot = 0
        for h in reasons:
            v = int(r[ix[h]] or 0)
            cls[e][h] += v
            tot += v
        inst.append((tot, e, r[ix["Source"]].strip(), {h: int(r[ix[h]] or 0) for h in reasons}))
    print(f"=== {name[:110]}")
    allsamp = sum(sum(c.values()) for c in cls.values())
    top = sorted(cls, key=lambda e: -sum(cls[e].values()))[:nclass]
    for e in top:
        c = cls[e]
        tot = sum(c.values())
        print(f"exec={e:10d} ninstr={ninst[e]:4d} samples={tot:7d} ({100 * tot / max(allsamp, 1):4.1f}%) " +
              " ".join(f"{k.replace('stall_', '')}={v}" for k, v in c.most_common(5)))
    print("top instructions:")
    for tot, e, src, st in sorted(inst, key=lambda t: -t[0])[:ntop]:
        best = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"  {tot:7d} exec={e:9d} {src[:60]:60s} " + " ".join(f"{k.replace('stall_', '')}={v}" for k, v in best))


rows = list(csv.reader(open(sys.argv[1])))
for sec in list(sections(rows)):
    if sec["rows"]:
        summarise(sec["name"], sec["rows"], int(sys.argv[2]) if len(sys.argv) > 2 else 8,
                  int(sys.argv[3]) if len(sys.argv) > 3 else 12)
