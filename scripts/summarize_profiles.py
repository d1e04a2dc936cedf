"""Summarize a round's GPU evidence into profiles/ (committed):
  profiles/<tag>_ncu_summary.json   key ncu --set full metrics of the switch / GEMV / fused / prefill captures
  profiles/<tag>_launches.md        per-kernel share of a bench step from the ncu launch list
  profiles/ncu_switch_traffic.json  DRAM bytes per layer of the switch capture (bench.py roofline.traffic)
Usage: python scripts/summarize_profiles.py TAG [gpurun_out]"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")][:80]}
        for w in WANT:
            # tolerate metric-name variants across ncu versions
            cands = [i for i, name in enumerate(h) if name == w]
            if cands:
                rec[w] = f"{r[cands[0]]} {u[cands[0]]}".strip()
        recs.append(rec)
    return recs


summary = {}
for name in ("switch", "gemv", "fused", "prefill"):
    rep = os.path.join(src, f"{name}_{tag}.ncu-rep")
    if os.path.exists(rep):
        summary[name] = raw(rep)
with open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w") as f:
    json.dump(summary, f, indent=1)

# traffic per layer of the switch capture (scripts/prof_kernels.py --layers 4)
if "switch" in summary and summary["switch"]:
    rec = summary["switch"][0]

    def gb(v):
        x, unit = v.split()[0], v.split()[1] if len(v.split()) > 1 else "byte"
        x = float(x.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    tot = gb(rec["dram__bytes_read.sum"]) + gb(rec["dram__bytes_write.sum"])
    with open(os.path.join(prof, "ncu_switch_traffic.json"), "w") as f:
        kname = rec["kernel"]
        json.dump({"config": "llama2-7b", "switch_impl": "tc", "capture_layers": 4, "round_tag": tag,
                   "kernel": kname, "switch_kernel": 3 if "switch_fc" in kname else None,
                   "dram_bytes_capture": tot, "dram_bytes_per_layer": tot / 4,
                   "note": "ncu --set full of the switch kernel (second pass: Eq. 10 fused switch) on the 7B "
                           "shape with 4 layers (identical per-matrix tiles); bench.py scales per layer x layers"},
                  f, indent=1)

# launch list shares
lfile = os.path.join(src, f"launches_{tag}.csv")
if os.path.exists(lfile):
    rows = list(csv.reader(open(lfile)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg, cnt = defaultdict(float), defaultdict(int)
    for r in data:
        k = r[ik].split("(")[0]
        agg[k] += float(r[iv].replace(",", ""))
        cnt[k] += 1
    tot = sum(agg.values())
    with open(os.path.join(prof, f"{tag}_launches.md"), "w") as f:
        f.write(f"# Launch list {tag}: `ncu --metrics gpu__time_duration.sum --clock-control none` over the bench's "
                f"2 timed decode tokens (cold-cache, serialised: compare shares)\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k in sorted(agg, key=lambda x: -agg[x]):
            f.write(f"| `{k}` | {cnt[k]} | {agg[k] / 1e6:.3f} | {agg[k] / tot * 100:.1f}% |\n")
    print(open(os.path.join(prof, f"{tag}_launches.md")).read())
print(json.dumps(summary, indent=1)[:3000])
