"""Text summary of an ncu --set full report (`ncu -i X.ncu-rep --page details --csv`): the
SOL, memory, compute, warp-state, launch and occupancy sections per kernel, plus DRAM bytes
from the raw page (development aid for profiles/)."""
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Warp State Statistics", "Launch Statistics", "Occupancy")
rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit")}
rr = list(csv.reader(io.StringIO(raw)))
rh = rr[0]
# pipe utilisation and traffic counters quoted in DESIGN.md / the bench line
EXTRA = ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
         "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
         "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
         "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors.sum", "lts__t_bytes.sum",
         "sm__cycles_elapsed.avg")
extra = {}
for r in rr[2:]:
    d = dict(zip(rh, r))
    if "ID" in d:
        extra[d["ID"]] = [(k, d[k], rr[1][rh.index(k)]) for k in EXTRA if k in d and d[k] != ""]
dram = {}
for r in rr[2:]:
    d = dict(zip(rh, r))
    try:
        dram[d["ID"]] = (float(d.get("dram__bytes_read.sum", "0").replace(",", "")),
                         float(d.get("dram__bytes_write.sum", "0").replace(",", "")), rr[1][rh.index("dram__bytes_read.sum")])
    except (KeyError, ValueError):
        pass
print(title)
cur = None
for r in rows[1:]:
    if r[ix["Section Name"]] not in SECTIONS:
        continue
    if r[ix["ID"]] != cur:
        cur = r[ix["ID"]]
        print(f"\n== launch {cur}: {r[ix['Kernel Name']][:110]}")
        if cur in dram:
            rd, wr, unit = dram[cur]
            print(f"  [raw] dram__bytes_read.sum + dram__bytes_write.sum: {rd:.4g} + {wr:.4g} {unit}")
        for k, v, u in extra.get(cur, []):
            print(f"  [raw] {k}: {v} {u}")
    print(f"  [{r[ix['Section Name']]}] {r[ix['Metric Name']]}: {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
