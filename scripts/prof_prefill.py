"""ncu target: one lsw_prefill_group call per GEMV group (7B widths, one layer,
512 tokens) -- the LoRA-down GEMM, the Z build and the dense + LoRA-up GEMM."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b").with_(n_layers=1)
T = 512
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl="tc")
X1 = synth.gen_x1(cfg, T, "cuda")
idx = torch.empty(T, cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(T, cfg.top_k, dtype=torch.float32, device="cuda")
for t in range(T):
    sw.router_topk(X1[t], idx[t], gate[t])
for gi, grp in enumerate(synth.GROUPS):
    d_in = cfg.kind_shape(grp[0])[1]
    rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
    X = torch.randn(T, d_in, device="cuda").to(torch.bfloat16)
    Y = torch.empty(T, rows, device="cuda")
    sw.prefill_group(0, gi, X, idx, gate, Y)
torch.cuda.synchronize()
print("done", sw.device_status())
