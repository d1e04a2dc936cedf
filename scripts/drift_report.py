"""Weight drift after T fused switches and after T merge/unmerge cycles
(north_star; R22), GPU (through the C ABI) and oracle side by side,
on sampled rows of every adapted kind of a few layers (row sampling is exact,
O9).  Writes one JSON object (stdout and --out).

  (i)  switch : T tokens of Alg. 1 (router -> fused switch); at T compare the
       stored weights with the exact P + DeltaW(d_T): rel. Frobenius drift,
       max-abs, fraction outside allclose(1e-2, 2e-2); GPU-vs-oracle divergence.
  (ii) cycles : T x (merge d_t; unmerge d_t) from the pristine weights; drift
       measured against P.
Expected: bf16 drift ~ eps1*sqrt(T) ~ 5e-2 for (i), ~3e-2 for
(ii) at rho = 0.25; GPU/oracle drift ratio ~ 1.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


def rows_for(d_out, seed, n):
    g = np.random.default_rng(seed)
    base = {0, 1, 127, 128, d_out - 1}
    base |= set(g.choice(d_out, size=min(n, d_out), replace=False).tolist())
    return sorted(r for r in base if 0 <= r < d_out)


def stats(W, ref):
    d = W - ref
    return {"rel_fro": float(np.linalg.norm(d) / np.linalg.norm(ref)), "max_abs": float(np.abs(d).max()),
            "frac_fail": float(np.mean(np.abs(d) > 1e-2 + 2e-2 * np.abs(ref)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama2-7b")
    ap.add_argument("--tokens", type=int, default=1000)
    ap.add_argument("--rows", type=int, default=16)
    ap.add_argument("--layers", default="0,15,31")
    ap.add_argument("--impl", default="auto")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.get_config(a.config)
    layers = [int(x) for x in a.layers.split(",") if int(x) < cfg.n_layers]
    store = "bf16" if cfg.dtype == "bf16" else "f32"
    scale = cfg.alpha / cfg.rank
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl=a.impl)
    rows = {kd: rows_for(cfg.kind_shape(kd)[0], 11 + i, a.rows) for i, kd in enumerate(synth.KINDS)}
    keys = [(kd, l) for kd in synth.KINDS for l in layers]
    P = {k: f64(W[k[0]][k[1]][rows[k[0]]]) for k in keys}
    An = {k: f64(A[k[0]][k[1]]) for k in keys}
    Bn = {k: f64(B[k[0]][k[1]][:, rows[k[0]], :]) for k in keys}
    Wg = f64(router)
    X1 = synth.gen_x1(cfg, a.tokens, "cuda")
    X1h = f64(X1)
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    out = {"config": cfg.name, "tokens": a.tokens, "impl": sw.info()["switch_impl"], "store": store,
           "rows_per_matrix": {kd: len(rows[kd]) for kd in synth.KINDS}, "layers": layers,
           "rho": synth.RHO}

    # ---------------- (i) fused switches
    orc = O.OracleModel(Wg, P, An, Bn, cfg.top_k, cfg.alpha, cfg.rank, store)
    t0 = time.time()
    same_prev = 0
    union = []
    prev_set = None
    for t in range(a.tokens):
        sw.router_topk(X1[t], idx, gate)
        sw.merge_all_layers(idx, gate)
        io, go, _ = orc.route(X1h[t])
        orc.merge_all_layers((io.tolist(), go.tolist()))
        s = set(io.tolist())
        if prev_set is not None:
            same_prev += s == prev_set
            union.append(len(s | prev_set))
        prev_set = s
        if t % 100 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    gpu_idx = idx.cpu().tolist()
    assert gpu_idx == io.tolist(), "router diverged"
    cur = (io.tolist(), go.tolist())
    agg = {"gpu_vs_exact": [], "orc_vs_exact": [], "gpu_vs_orc": []}
    Wg_all, Wo_all, We_all = [], [], []
    for k in keys:
        Wgpu = f64(W[k[0]][k[1]][rows[k[0]]])
        exact = P[k] + O.delta(An[k], Bn[k], O.coef_list(cur, None, scale))
        Wg_all.append(Wgpu.ravel())
        Wo_all.append(orc.W[k].ravel())
        We_all.append(exact.ravel())
    Wg_all, Wo_all, We_all = map(np.concatenate, (Wg_all, Wo_all, We_all))
    out["switch"] = {"gpu_vs_exact": stats(Wg_all, We_all), "oracle_vs_exact": stats(Wo_all, We_all),
                     "gpu_vs_oracle": stats(Wg_all, Wo_all),
                     "frac_tokens_same_experts_as_prev": same_prev / max(1, a.tokens - 1),
                     "mean_union_size": float(np.mean(union)) if union else None,
                     "seconds": time.time() - t0}
    out["switch"]["drift_ratio_gpu_over_oracle"] = (out["switch"]["gpu_vs_exact"]["rel_fro"] /
                                                    out["switch"]["oracle_vs_exact"]["rel_fro"])
    sw.unmerge_all_layers()
    torch.cuda.synchronize()
    # restore the pristine weights on the GPU for part (ii)
    for kd in synth.KINDS:
        for l in range(cfg.n_layers):
            W[kd][l].copy_(synth.gen_W(cfg, kd, l, "cuda"))
    sw.close()
    sw = H.make_switch(cfg, W, A, B, router, impl=a.impl)

    # ---------------- (ii) merge / unmerge cycles
    orc2 = O.OracleModel(Wg, P, An, Bn, cfg.top_k, cfg.alpha, cfg.rank, store)
    t0 = time.time()
    for t in range(a.tokens):
        sw.router_topk(X1[t], idx, gate)
        sw.merge_all_layers(idx, gate)
        sw.unmerge_all_layers()
        io, go, _ = orc2.route(X1h[t])
        orc2.merge_all_layers((io.tolist(), go.tolist()))
        orc2.unmerge_all_layers()
        if t % 100 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    Wg_all, Wo_all, P_all = [], [], []
    for k in keys:
        Wg_all.append(f64(W[k[0]][k[1]][rows[k[0]]]).ravel())
        Wo_all.append(orc2.W[k].ravel())
        P_all.append(P[k].ravel())
    Wg_all, Wo_all, P_all = map(np.concatenate, (Wg_all, Wo_all, P_all))
    out["cycles"] = {"gpu_vs_pristine": stats(Wg_all, P_all), "oracle_vs_pristine": stats(Wo_all, P_all),
                     "gpu_vs_oracle": stats(Wg_all, Wo_all), "seconds": time.time() - t0}
    out["cycles"]["drift_ratio_gpu_over_oracle"] = (out["cycles"]["gpu_vs_pristine"]["rel_fro"] /
                                                    out["cycles"]["oracle_vs_pristine"]["rel_fro"])
    assert sw.device_status() == 0
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
