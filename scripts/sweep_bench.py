"""BASELINE configs[4]: merge-kernel sweep on the Llama-2-7B shape, rank 4..64 x
top-k 1..4 x experts 4..16 (k <= N), GB/s of the fused switch and of a plain
merge vs the roofline max(bytes / HBM peak, FLOPs / tensor peak).

The backbone W is generated once; adapters per (N, r); one ctx per cell.
Writes one JSON object per cell (stdout, and --out as a JSON list)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--layers", type=int, default=0, help="0 = full 32 layers")
ap.add_argument("--ranks", default="4,8,16,32,64")
ap.add_argument("--experts", default="4,8,16")
ap.add_argument("--topk", default="1,2,3,4")
ap.add_argument("--out", default="")
a = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6452.8, "bf16_tflops_sustained": 1425.9}
hbm, tc = peaks["hbm_gbs"], peaks.get("bf16_tflops_sustained", 1425.9)
base = synth.get_config("llama2-7b")
if a.layers:
    base = base.with_(n_layers=a.layers)
W, _, _, router0 = H.build_weights(base, "cuda", kinds=synth.KINDS)
rows = []
for n in [int(x) for x in a.experts.split(",")]:
    for r in [int(x) for x in a.ranks.split(",")]:
        cfg_nr = base.with_(name=f"sweep-n{n}-r{r}", n_experts=n, rank=r, top_k=min(2, n))
        A = {kd: torch.empty(base.n_layers, n, r, base.kind_shape(kd)[1], dtype=torch.bfloat16, device="cuda")
             for kd in synth.KINDS}
        B = {kd: torch.empty(base.n_layers, n, base.kind_shape(kd)[0], r, dtype=torch.bfloat16, device="cuda")
             for kd in synth.KINDS}
        for kd in synth.KINDS:
            for l in range(base.n_layers):
                A[kd][l].copy_(synth.gen_A(cfg_nr, kd, l, "cuda"))
                B[kd][l].copy_(synth.gen_B(cfg_nr, kd, l, "cuda"))
        router = synth.gen_router(cfg_nr, "cuda")
        for k in [int(x) for x in a.topk.split(",")]:
            if k > n:
                continue
            cfg = cfg_nr.with_(name=f"sweep-n{n}-r{r}-k{k}", top_k=k)
            X1 = synth.gen_x1(cfg, a.iters + 2, "cuda")
            idx = torch.empty(k, dtype=torch.int32, device="cuda")
            gate = torch.empty(k, dtype=torch.float32, device="cuda")
            rec = {"cell": cfg.name, "N": n, "r": r, "k": k}
            try:
                sw = H.make_switch(cfg, W, A, B, router, impl="auto")
            except Exception as e:  # noqa: BLE001
                rec["error"] = str(e)
                print(json.dumps(rec), flush=True)
                rows.append(rec)
                continue
            sw.router_topk(X1[0], idx, gate)
            sw.merge_all_layers(idx, gate)
            ms, terms = [], []
            prev = set(idx.cpu().tolist())
            for t in range(1, a.iters + 1):
                sw.router_topk(X1[t], idx, gate)
                cur = set(idx.cpu().tolist())
                terms.append(len(cur | prev))
                prev = cur
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sw.merge_all_layers(idx, gate)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            sw.unmerge_all_layers()
            e1.record()
            sw.merge_all_layers(idx, gate)
            e2.record()
            torch.cuda.synchronize()
            merge_ms = e1.elapsed_time(e2)
            sw.unmerge_all_layers()
            torch.cuda.synchronize()
            tb = H.token_bytes(cfg)
            med = statistics.median(ms)
            mean_terms = statistics.mean(terms)
            # algorithmic bytes/flops at the realized (compacted) term count
            s = cfg.elem_bytes
            w_el = tb["w_elems"]
            io = sum((cfg.kind_shape(kd)[0] + cfg.kind_shape(kd)[1]) for kd in synth.KINDS) * cfg.n_layers
            sw_bytes_real = 2 * s * w_el + s * mean_terms * r * io
            sw_flops_real = 2 * mean_terms * r * w_el
            roof_ms = max(sw_bytes_real / (hbm * 1e9), sw_flops_real / (tc * 1e12)) * 1e3
            rec.update({"impl": sw.info()["switch_impl"], "switch_ms": round(med, 4),
                        "switch_GBps_2k": round(tb["switch"] / (med * 1e-3) / 1e9, 1),
                        "mean_terms": mean_terms,
                        "switch_GBps_realized": round(sw_bytes_real / (med * 1e-3) / 1e9, 1),
                        "switch_frac_of_roofline": round(roof_ms / med, 4),
                        "merge_ms": round(merge_ms, 4),
                        "merge_GBps": round(tb["merge"] / (merge_ms * 1e-3) / 1e9, 1),
                        "bound": "tensor" if sw_flops_real / (tc * 1e12) > sw_bytes_real / (hbm * 1e9) else "hbm"})
            assert sw.device_status() == 0
            sw.close()
            print(json.dumps(rec), flush=True)
            rows.append(rec)
        del A, B
        torch.cuda.empty_cache()
if a.out:
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)
