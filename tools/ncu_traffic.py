#!/usr/bin/env python
"""Extract the roofline/traffic numbers of one ncu capture (run here, on the
CPU box) into profiles/traffic_<name>.json, which bench.py's roofline reads:

  python tools/ncu_traffic.py REPORT.ncu-rep NAME "how it was captured"
"""
import csv
import io
import json
import subprocess
import sys

rep, name, how = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, vals = rows[0], rows[1], rows[2]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def get(k):
    i = hdr.index(k)
    v = float(vals[i].replace(",", ""))
    return v * SCALE.get(units[i], 1.0)


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
out = {"kernel": vals[hdr.index("Kernel Name")][:80], "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": int(rd + wr), "duration_s_ncu": get("gpu__time_duration.sum"),
       "warp_instructions": get("smsp__inst_executed.sum"),
       "active_threads_per_inst": get("smsp__thread_inst_executed_per_inst_executed.ratio"),
       "sectors_per_request": get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
       / max(1.0, get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")),
       "source": f"ncu --set full --clock-control none ({how}); report {rep}"}
for k in ("lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__issue_active.avg.pct_of_peak_sustained_active"):
    if k in hdr:
        out[k] = get(k)
with open(f"profiles/traffic_{name}.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
