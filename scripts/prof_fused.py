"""ncu target: the plain sweep-order switch and the fused switch + decode on a
4-layer slice of the 7B shape (identical per-layer tiles).  Launch order of
switch_fc_kernel: 1 merge, 2 switch (sweep order), 3-4 fused tokens."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b").with_(n_layers=4)
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl="tc")
X1 = synth.gen_x1(cfg, 8, "cuda")
xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
ys = torch.empty(sw.info()["ys_elems"], device="cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
sw.router_topk(X1[0], idx, gate)
sw.merge_all_layers(idx, gate)
sw.router_topk(X1[1], idx, gate)
sw.merge_all_layers(idx, gate)
sw.decode_token_fused(X1[2], xs, ys, idx, gate)
sw.decode_token_fused(X1[3], xs, ys, idx, gate)
torch.cuda.synchronize()
print("done", sw.device_status())
