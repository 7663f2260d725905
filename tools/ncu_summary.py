"""Summarise an ncu --set full capture into the JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/ncu_full_x.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    # register spills actually executed (local-memory traffic)
    "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_local_op_st.sum"]
STALL = "smsp__average_warps_issue_stalled_"

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    entry = {"kernel": d.get("Kernel Name", "")}
    for m in METRICS:
        if m in d:
            try:
                entry[m] = float(d[m].replace(",", ""))
            except ValueError:
                entry[m] = d[m]
    stalls = {}
    for k, v in d.items():
        if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
            try:
                stalls[k[len(STALL):-len("_per_issue_active.ratio")]] = \
                    float(v.replace(",", ""))
            except ValueError:
                pass
    entry["top_stalls_per_issue"] = dict(
        sorted(stalls.items(), key=lambda kv: -kv[1])[:4])
    out.append(entry)
print(json.dumps({"source": sys.argv[1].split("/")[-1],
                  "units": {m: units[hdr.index(m)] for m in METRICS
                            if m in hdr},
                  "launches": out}, indent=1))
