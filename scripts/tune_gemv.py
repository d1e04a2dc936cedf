"""Time the decode GEMV groups at a BASELINE shape (variant from LSW_GEMV=ldg|bulk,
read once per process).  Prints per-group median us, GB/s (algorithmic bytes,
read-only) and the whole-token GEMV time (4 groups x L layers, stream order)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama2-7b")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = synth.get_config(a.config)
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl="auto")
xs = synth.gen_xs(cfg, "cuda")
res = {"variant": os.environ.get("LSW_GEMV", "bulk")}
for gi, grp in enumerate(synth.GROUPS):
    n = sum(cfg.kind_shape(k)[0] for k in grp)
    d_in = cfg.kind_shape(grp[0])[1]
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    ts = []
    for it in range(a.iters):
        l = it % cfg.n_layers
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sw.decode_group(l, gi, xs[(l, gi)], y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    med = statistics.median(ts)
    nbytes = n * d_in * cfg.elem_bytes + d_in * cfg.elem_bytes + 4 * n
    res["+".join(grp)] = {"us": round(med * 1e3, 2), "GBps": round(nbytes / (med * 1e-3) / 1e9, 1)}
# whole token of GEMVs back to back
xs_p = H.pack_xs(cfg, xs)
info = sw.info()
ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
tok = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    xo = yo = 0
    for l in range(cfg.n_layers):
        for gi, grp in enumerate(synth.GROUPS):
            d_in = cfg.kind_shape(grp[0])[1]
            n = sum(cfg.kind_shape(k)[0] for k in grp)
            sw.decode_group(l, gi, xs_p[xo:xo + d_in], ys[yo:yo + n])
            xo += d_in
            yo += n
    e1.record()
    torch.cuda.synchronize()
    tok.append(e0.elapsed_time(e1))
tb = H.token_bytes(cfg)
med = statistics.median(tok)
res["groups_gemv_ms"] = round(med, 4)
res["groups_gemv_GBps"] = round(tb["gemv"] / (med * 1e-3) / 1e9, 1)
# whole-token launch (lsw_decode_all_layers: one persistent GEMV when tp_size == 1)
tok = []
for rep in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sw.decode_all_layers(xs_p, ys)
    e1.record()
    torch.cuda.synchronize()
    tok.append(e0.elapsed_time(e1))
med = statistics.median(tok)
res["token_gemv_ms"] = round(med, 4)
res["token_gemv_GBps"] = round(tb["gemv"] / (med * 1e-3) / 1e9, 1)
res["env"] = {k: v for k, v in os.environ.items() if k.startswith("LSW_")}
print(json.dumps(res), flush=True)
