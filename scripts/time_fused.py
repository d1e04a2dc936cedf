"""Tuning: decode ms/token, separate (lsw_decode_token) vs fused (lsw_decode_token_fused)."""
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
X1 = synth.gen_x1(cfg, 24, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
def t(fn, n=10):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): fn(3 + i)
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n, 4)
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("LSW_")},
       "separate_ms": t(lambda i: sw.decode_token(X1[i], xs, ys, idx, gate)),
       "fused_ms": t(lambda i: sw.decode_token_fused(X1[i], xs, ys, idx, gate))}
print(json.dumps(res))
