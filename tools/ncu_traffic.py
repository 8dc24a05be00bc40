"""Summarise an `ncu --set full` report: per kernel launch, duration and DRAM bytes (read + write).

    python tools/ncu_traffic.py report.ncu-rep [--config C2 --json profiles/traffic.json --issue profiles/issue.json]

--issue also records, per kernel, the issue-active, SM-throughput and tensor-pipe percentages and the shared-memory
data-pipe utilisation (LSU + tensor-core wavefronts): the numbers bench.py attaches as roofline.ncu_utilisation.
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
ap.add_argument("--issue")
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
    util = {}
    for key, name in (("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                      ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                      ("tensor_pipe_active_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                      ("smem_lsu_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                      ("smem_tc_pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")):
        if name in col:
            util[key] = num(name)
    res.append({"kernel": r[col["Kernel Name"]][:80], "ms": dur, "dram_read_B": rd, "dram_write_B": wr,
                "dram_B": rd + wr, "dram_GBps": (rd + wr) / (dur * 1e-3) / 1e9 if dur else None, **util})
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
if a.issue and a.config:
    try:
        with open(a.issue) as f:
            iss = json.load(f)
    except OSError:
        iss = {}
    iss[a.config] = {x["kernel"].split("(")[0].split("<")[0].split()[-1]:
                     {k: x[k] for k in ("issue_active_pct", "sm_throughput_pct", "tensor_pipe_active_pct", "smem_lsu_pct",
                                        "smem_tc_pct") if k in x} for x in res}
    with open(a.issue, "w") as f:
        json.dump(iss, f, indent=1)
