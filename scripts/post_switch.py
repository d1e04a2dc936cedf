"""Decode GEMVs of a token right after the switch vs on their own (7B): CUDA
events around lsw_decode_all_layers (a) back to back with nothing before,
(b) right behind a switch launch, (c) behind a switch followed by a host
sleep (L2 write-backs drained, clocks settled).  Shows what the switch
leaves behind for the GEMVs."""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b")
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl="tc")
xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
ys = torch.empty(sw.info()["ys_elems"], device="cuda")
X1 = synth.gen_x1(cfg, 64, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


res = {"alone": [], "after_switch": [], "after_switch_sleep": [], "switch": []}
for t in range(24):
    sw.router_topk(X1[t], idx, gate)
    a, b, c = ev(), ev(), ev()
    a.record()
    sw.merge_all_layers(idx, gate)
    b.record()
    sw.decode_all_layers(xs, ys)
    c.record()
    torch.cuda.synchronize()
    if t >= 4:
        res["switch"].append(a.elapsed_time(b))
        res["after_switch"].append(b.elapsed_time(c))
    sw.router_topk(X1[t + 30], idx, gate)
    sw.merge_all_layers(idx, gate)
    torch.cuda.synchronize()
    time.sleep(0.01)
    a, b = ev(), ev()
    a.record()
    sw.decode_all_layers(xs, ys)
    b.record()
    torch.cuda.synchronize()
    if t >= 4:
        res["after_switch_sleep"].append(a.elapsed_time(b))
    a, b = ev(), ev()
    a.record()
    sw.decode_all_layers(xs, ys)
    b.record()
    torch.cuda.synchronize()
    if t >= 4:
        res["alone"].append(a.elapsed_time(b))
print({k: round(statistics.median(v), 4) for k, v in res.items()})
