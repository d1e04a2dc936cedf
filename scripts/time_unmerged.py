"""Tuning: whole-token unmerged decode time (decode_all_layers_unmerged) under
LSW_UNMERGED_FLAGS probes, next to the merged GEMVs (decode_all_layers)."""
import os, statistics, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2405_17741_b200 import harness as H
cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b")
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router)
xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
ys = torch.empty(sw.info()["ys_elems"], device="cuda")
X1 = synth.gen_x1(cfg, 4, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
sw.router_topk(X1[0], idx, gate)
def t(fn, n=8):
    ms = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 4)
res = {"merged_gemvs": t(lambda: sw.decode_all_layers(xs, ys))}
for f in ["0", "4"]:
    os.environ["LSW_UNMERGED_FLAGS"] = f
    res["unmerged_flags" + f] = t(lambda: sw.decode_all_layers_unmerged(xs, ys, idx, gate))
os.environ.pop("LSW_UNMERGED_FLAGS", None)
print(json.dumps(res))
