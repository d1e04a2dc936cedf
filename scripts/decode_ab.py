"""A/B of the decode paths of two liblsw builds on one box (7B): per token,
the merged-weight GEMVs (lsw_decode_all_layers) and the unmerged decode
(router + lsw_decode_all_layers_unmerged).  Usage:
python scripts/decode_ab.py [--lib path] config [option=value ...] (variant
options, include/lsw_debug.h, for the ctx)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def med(fn, n=30):
    ms = []
    for _ in range(n + 5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ms = sorted(ms[5:])
    return ms[len(ms) // 2]


def main():
    label = "new"
    if sys.argv[1] == "--lib":
        binding._LIB = binding.load_library(sys.argv[2], strict=False)
        label = os.path.basename(sys.argv[2])
        del sys.argv[1:3]
    cfg = synth.get_config(sys.argv[1])
    opts = dict(kv.split("=") for kv in sys.argv[2:])
    if opts:
        label += " " + ",".join(sys.argv[2:])
    W, A, B, router = H.build_weights(cfg, "cuda")
    with binding.options(**opts):
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    ys = torch.empty(sw.info()["ys_elems"], device="cuda")
    X1 = synth.gen_x1(cfg, 2, "cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    sw.router_topk(X1[0], idx, gate)
    un = med(lambda: (sw.router_topk(X1[0], idx, gate), sw.decode_all_layers_unmerged(xs, ys, idx, gate)))
    gm = med(lambda: sw.decode_all_layers(xs, ys))
    print(f"{label}: gemv {gm:.3f} ms  unmerged {un:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
