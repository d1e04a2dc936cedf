"""Time the all-layer switch kernel at a BASELINE shape under variant options
(include/lsw_debug.h lsw_debug_set_option, read at lsw_create).  Prints one
line per setting: median switch GB/s (algorithmic bytes) and fraction of the
measured copy peak.  Usage: python scripts/tune_switch.py [--config llama2-7b]
SETTING... where SETTING is like 'tc_kernel=pt,tc_chunk=32,fc_wrm=0' (probe
options need a -DLSW_TUNING build)."""
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
ap.add_argument("--layers", type=int, default=0)
ap.add_argument("--iters", type=int, default=12)
ap.add_argument("--impl", default="tc")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--rank", type=int, default=0, help="override the config's LoRA rank (sweep cells)")
ap.add_argument("--topk", type=int, default=0, help="override the config's top-k (sweep cells)")
ap.add_argument("--lib", default="", help="load this liblsw.so instead of the package's (A/B of two builds)")
ap.add_argument("settings", nargs="*", default=["", "tc_chunk=32", "tc_chunk=64"])
a = ap.parse_args()
from paper_2405_17741_b200 import binding as _B  # noqa: E402
if a.lib:
    _B._LIB = _B.load_library(a.lib, strict=False)
cfg = synth.get_config(a.config)
if a.layers:
    cfg = cfg.with_(n_layers=a.layers)
if a.rank:
    cfg = cfg.with_(rank=a.rank)
if a.topk:
    cfg = cfg.with_(top_k=a.topk)
W, A, B, router = H.build_weights(cfg, "cuda")
tb = H.token_bytes(cfg)
X1 = synth.gen_x1(cfg, a.iters + 4, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6452.8
for setting in [x for _ in range(a.repeat) for x in a.settings]:
    _B.set_option(None)
    opts = dict(kv.split("=") for kv in setting.split(",") if kv)
    for k, v in opts.items():
        _B.set_option(k, v)
    try:
        sw = H.make_switch(cfg, W, A, B, router, impl=a.impl)
    except Exception as e:  # noqa: BLE001  (no plan for this shape under these knobs)
        print(json.dumps({"setting": setting, "error": str(e)[:120]}), flush=True)
        continue
    probe = opts.get("tc_probe", "0") == "1"
    sw.router_topk(X1[0], idx, gate)
    sw.merge_all_layers(idx, gate)
    ms = []
    for t in range(1, a.iters + 1):
        sw.router_topk(X1[t], idx, gate)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sw.merge_all_layers(idx, gate)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    sw.unmerge_all_layers()
    torch.cuda.synchronize()
    med = statistics.median(ms)
    nbytes = 2 * cfg.elem_bytes * tb["w_elems"] if probe else tb["switch"]
    gbs = nbytes / (med * 1e-3) / 1e9
    print(json.dumps({"setting": setting, "impl": sw.info()["switch_impl"], "ms": round(med, 4),
                      "GBps": round(gbs, 1), "frac": round(gbs / peak, 4), "min_ms": round(min(ms), 4)}), flush=True)
    assert sw.device_status() == 0
    sw.close()
