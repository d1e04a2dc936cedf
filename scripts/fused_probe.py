"""Where the fused switch + decode spends its time (7B): needs the tuning build
(python paper_2405_17741_b200/build.py --tuning), whose probe options give
deliberately WRONG results.  Times per token (CUDA events, 30 tokens after 5):
  fused            lsw_decode_token_fused as shipped
  fused_nowait     fc_fused_probe=4: no segment waits (decoder dependency dropped)
  fused_nogemv     fc_fused_probe=8: decoder-order switch without the GEMV epilogue
  fused_bare       fc_fused_probe=12
  fused_wstream    fc_fused_probe=5: the W stream alone in decoder order, no waits
  switch           the plain sweep-order switch (lsw_merge_all_layers)
  switch_wstream   tc_probe=1: the W stream alone (load + store, no math)
JSON to stdout."""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    X1 = synth.gen_x1(cfg, 40, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    out = {"config": name}
    cases = [("fused", {}, True), ("fused_nowait", {"fc_fused_probe": 4}, True),
             ("fused_nogemv", {"fc_fused_probe": 8}, True), ("fused_bare", {"fc_fused_probe": 12}, True),
             ("fused_wstream", {"fc_fused_probe": 5}, True),
             ("switch", {}, False), ("switch_wstream", {"tc_probe": 1}, False)]
    for label, opts, fused in cases:
        with binding.options(**opts):
            sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        info = sw.info()
        ys = torch.empty(info["ys_elems"], device="cuda")
        idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
        ms = []
        for t in range(35):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if fused:
                a.record()
                sw.decode_token_fused(X1[t], xs, ys, idx, gate)
                b.record()
            else:
                sw.router_topk(X1[t], idx, gate)
                a.record()
                sw.merge_all_layers(idx, gate)
                b.record()
            torch.cuda.synchronize()
            if t >= 5:
                ms.append(a.elapsed_time(b))
        ms.sort()
        out[label] = {"median_ms": ms[len(ms) // 2], "min_ms": ms[0]}
        sw.unmerge_all_layers()
        torch.cuda.synchronize()
        sw.close()
        print(label, out[label], file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
