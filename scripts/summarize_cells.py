"""Key ncu --set full metrics of the per-cell switch captures (scripts/gpu_ncu_cells.sh)
-> profiles/<tag>_ncu_cells.json.  Usage: python scripts/summarize_cells.py TAG [gpurun_out]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
out = {}
for name in sorted(os.listdir(src)):
    if not (name.startswith("cell_") and name.endswith(".ncu-rep")):
        continue
    txt = subprocess.run(["ncu", "-i", os.path.join(src, name), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, r = rows[0], rows[1], rows[2]
    rec = {"kernel": r[h.index("Kernel Name")]}
    for w in WANT:
        if w in h:
            i = h.index(w)
            rec[w] = f"{r[i]} {u[i]}".strip()
    out[name[len("cell_"):-len(".ncu-rep")]] = rec
with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_cells.json"), "w") as f:
    json.dump(out, f, indent=1)
for k, v in out.items():
    print(k, v["kernel"][:40], {a.split("__")[1][:28]: b for a, b in v.items() if a != "kernel"})
