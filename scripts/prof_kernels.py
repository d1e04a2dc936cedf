"""Small driver for ncu: the Llama-2-7B per-matrix shapes with fewer layers
(identical tiles per matrix, so per-launch behaviour matches the full model
while ncu's save/restore of the in-place W stays small).  Runs a few decode
tokens through lsw_decode_token."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama2-7b")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--tokens", type=int, default=4)
ap.add_argument("--impl", default="auto")
ap.add_argument("--rank", type=int, default=0, help="override the config's LoRA rank (sweep cells)")
ap.add_argument("--topk", type=int, default=0, help="override the config's top-k (sweep cells)")
a = ap.parse_args()
cfg = synth.get_config(a.config).with_(n_layers=a.layers)
if a.rank:
    cfg = cfg.with_(rank=a.rank)
if a.topk:
    cfg = cfg.with_(top_k=a.topk)
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl=a.impl)
X1 = synth.gen_x1(cfg, a.tokens, "cuda")
xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
info = sw.info()
ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
for t in range(a.tokens):
    sw.decode_token(X1[t], xs, ys, idx, gate)
torch.cuda.synchronize()
print("ok", info)
