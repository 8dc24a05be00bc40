"""Summarise an `ncu --set full` report: per kernel launch, duration and DRAM bytes (read + write).

    python tools/ncu_traffic.py report.ncu-rep [--config C2 --json profiles/traffic.json]
"""
import argparse
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--config")
ap.add_argument("--json")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
col = {name: i for i, name in enumerate(h)}
res = []
for r in rows[2:]:
    def num(name):
        v = r[col[name]].replace(",", "")
        try:
            return float(v)
        except ValueError:
            return None
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr *= scale.get(units[col["dram__bytes_write.sum"]], 1)
    dur = num("gpu__time_duration.sum") * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
        units[col["gpu__time_duration.sum"]], 1.0)
    res.append({"kernel": r[col["Kernel Name"]][:80], "ms": dur, "dram_read_B": rd, "dram_write_B": wr,
                "dram_B": rd + wr, "dram_GBps": (rd + wr) / (dur * 1e-3) / 1e9 if dur else None})
for x in res:
    print(json.dumps(x))
if a.json and a.config:
    try:
        with open(a.json) as f:
            tr = json.load(f)
    except OSError:
        tr = {}
    tr[a.config] = {x["kernel"].split("(")[0].split("<")[0].split()[-1]: x["dram_B"] for x in res}
    with open(a.json, "w") as f:
        json.dump(tr, f, indent=1)
