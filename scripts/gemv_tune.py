"""Decode-GEMV variants on one token of GEMVs (lsw_decode_all_layers, 7B):
median ms over 30 tokens, each variant a fresh ctx over the same weights.
Usage: python scripts/gemv_tune.py [config] 'label:key=val,key=val' ..."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def main():
    name = sys.argv[1]
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    tb = H.token_bytes(cfg)["gemv"]
    out = {"config": name, "gemv_bytes": tb}
    for spec in sys.argv[2:] * 2:                       # every variant twice, interleaved
        label, _, kv = spec.partition(":")
        opts = dict(x.split("=") for x in kv.split(",") if x)
        with binding.options(**opts):
            sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        ys = torch.empty(sw.info()["ys_elems"], device="cuda")
        ms = []
        for t in range(35):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sw.decode_all_layers(xs, ys)
            b.record()
            torch.cuda.synchronize()
            if t >= 5:
                ms.append(a.elapsed_time(b))
        ms.sort()
        med = ms[len(ms) // 2]
        out.setdefault(label, []).append({"median_ms": med, "TBps": tb / med / 1e9})
        print(label, out[label][-1], file=sys.stderr, flush=True)
        sw.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
