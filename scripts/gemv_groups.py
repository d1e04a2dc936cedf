"""Decode-GEMV throughput per group type (q|k|v, o, gate|up, down): the same
group of every layer launched back to back (lsw_decode_group, PDL-chained as
in a token), median of 20 repetitions; GB/s of W bytes.  Shows which group
shape falls short of the read-stream rate.  --unmerged: the unmerged decode
(lsw_decode_group_unmerged, W pristine, LoRA terms in the same launch).
Usage: python scripts/gemv_groups.py [--unmerged] [config] [option=value ...]"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def main():
    unmerged = "--unmerged" in sys.argv
    if unmerged:
        sys.argv.remove("--unmerged")
    name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    opts = dict(kv.split("=") for kv in sys.argv[2:])
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    with binding.options(**opts):
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    out = {"config": name, "opts": opts, "unmerged": unmerged}
    idx = torch.tensor(list(range(cfg.top_k)), dtype=torch.int32, device="cuda")
    gate = torch.full((cfg.top_k,), 1.0 / cfg.top_k, dtype=torch.float32, device="cuda")
    for gi, grp in enumerate(synth.GROUPS):
        d_in = cfg.kind_shape(grp[0])[1]
        d_out = sum(cfg.kind_shape(k)[0] for k in grp)
        x = torch.randn(d_in, device="cuda").to(torch.bfloat16)
        y = torch.empty(d_out, device="cuda")
        ms = []
        for rep in range(25):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for layer in range(cfg.n_layers):
                if unmerged:
                    sw.decode_group_unmerged(layer, gi, x, y, idx, gate)
                else:
                    sw.decode_group(layer, gi, x, y)
            b.record()
            torch.cuda.synchronize()
            if rep >= 5:
                ms.append(a.elapsed_time(b))
        med = statistics.median(ms)
        nbytes = 2.0 * d_in * d_out * cfg.n_layers
        out["+".join(grp)] = {"ms": round(med, 4), "us_per_launch": round(1e3 * med / cfg.n_layers, 2),
                              "GBps": round(nbytes / (med * 1e-3) / 1e9, 1), "MB_per_launch": round(nbytes / cfg.n_layers / 1e6, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
