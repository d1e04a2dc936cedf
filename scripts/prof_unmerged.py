"""Profile helper: a few unmerged decode tokens (router + lsw_decode_all_layers_unmerged)."""
import os, sys
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
for t in range(3):
    sw.router_topk(X1[t], idx, gate)
    sw.decode_all_layers_unmerged(xs, ys, idx, gate)
torch.cuda.synchronize()
