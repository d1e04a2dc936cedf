"""Fused switch + decode variants (lsw_decode_token_fused, default 7B): median
ms per token over 30 tokens, each variant a fresh ctx over the same weights.
Usage: python scripts/fused_tune.py [config] 'label:key=val,key=val' ..."""
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
    if sys.argv[1] == "--lib":                  # A/B of two builds: --lib path config specs...
        lib = sys.argv[2]
        del sys.argv[1:3]
        binding._LIB = binding.load_library(lib, strict=False)
    name = sys.argv[1]
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    X1 = synth.gen_x1(cfg, 40, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    out = {"config": name}
    for spec in sys.argv[2:] * 2:
        label, _, kv = spec.partition(":")
        opts = dict(x.split("=") for x in kv.split(",") if x)
        try:
            with binding.options(**opts):
                sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        except binding.LswError as e:
            print(label, "unsupported", e, file=sys.stderr)
            continue
        ys = torch.empty(sw.info()["ys_elems"], device="cuda")
        idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
        ms = []
        for t in range(35):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sw.decode_token_fused(X1[t], xs, ys, idx, gate)
            b.record()
            torch.cuda.synchronize()
            if t >= 5:
                ms.append(a.elapsed_time(b))
        ms.sort()
        out.setdefault(label, []).append(ms[len(ms) // 2])
        print(label, ms[len(ms) // 2], file=sys.stderr, flush=True)
        sw.unmerge_all_layers()
        torch.cuda.synchronize()
        sw.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
