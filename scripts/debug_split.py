"""Multi-tile-per-CTA check of the tensor-core switch on the mini config
(LSW_TC_GRID small): run N switches, compare with the oracle, report."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, synth
from paper_2405_17741_b200 import harness as H
cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "mini")
W, A, B, router = H.build_weights(cfg, "cuda")
f64 = lambda t: t.detach().cpu().double().numpy()
P = {k: f64(W[k]) for k in synth.KINDS}
An = {k: f64(A[k]) for k in synth.KINDS}; Bn = {k: f64(B[k]) for k in synth.KINDS}
sw = H.make_switch(cfg, W, A, B, router, impl="tc")
print("info", sw.info(), flush=True)
X1 = synth.gen_x1(cfg, 6, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda"); gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
prev = None
for t in range(6):
    sw.router_topk(X1[t], idx, gate); sw.merge_all_layers(idx, gate)
    torch.cuda.synchronize()
    io, go, _ = O.router(f64(router), f64(X1[t]), cfg.top_k)
    cur = (io.tolist(), go.tolist())
    worst = 0
    for k in synth.KINDS:
        for l in range(cfg.n_layers):
            P[k][l] = O.switch(P[k][l], An[k][l], Bn[k][l], prev, cur, cfg.alpha / cfg.rank, "bf16")
            d = np.abs(f64(W[k][l]) - P[k][l]).max()
            worst = max(worst, d)
    prev = cur
    print(f"token {t}: max |gpu - oracle| = {worst:.3e}", flush=True)
