"""Prefill timing per GEMV group (7B widths, T tokens): lsw_prefill_group with
the token tile chosen per group (auto) or forced to 128 / 256 (variant option pf_tt), next to the same
dense products by torch.matmul (cuBLAS, reference only) -- JSON to stdout."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    extra = dict(kv.split("=") for kv in sys.argv[3:])       # variant options for every run
    cfg = synth.get_config(name).with_(n_layers=2)
    W, A, B, router = H.build_weights(cfg, "cuda")
    out = {"config": name, "T": T}
    X1 = synth.gen_x1(cfg, T, "cuda")
    for tt in (0, 128, 256):
        idx = torch.empty(T, cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(T, cfg.top_k, dtype=torch.float32, device="cuda")
        # the prefill plan is built at the first prefill call: inside the
        # options block, or the option would not reach it
        with binding.options(**({"pf_tt": tt} if tt else {}), **extra):
            sw = H.make_switch(cfg, W, A, B, router, impl="tc")
            for t in range(T):
                sw.router_topk(X1[t], idx[t], gate[t])
            d_in0 = cfg.kind_shape(synth.GROUPS[1][0])[1]
            rows0 = cfg.kind_shape(synth.GROUPS[1][0])[0]
            sw.prefill_group(1, 1, torch.zeros(T, d_in0, device="cuda", dtype=torch.bfloat16), idx, gate,
                             torch.empty(T, rows0, device="cuda"))
        res = {}
        for gi, grp in enumerate(synth.GROUPS):
            d_in = cfg.kind_shape(grp[0])[1]
            rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
            X = torch.randn(T, d_in, device="cuda").to(torch.bfloat16)
            Y = torch.empty(T, rows, device="cuda")
            ms = timed(lambda: sw.prefill_group(1, gi, X, idx, gate, Y))
            fl = 2.0 * T * rows * d_in
            res["+".join(grp)] = {"ms": ms, "dense_tflops": fl / ms / 1e9}
            if tt == 0:
                Wc = torch.cat([W[kd][1] for kd in grp])
                ms_ref = timed(lambda: torch.matmul(X, Wc.t(), out=None))
                res["+".join(grp)]["torch_matmul_bf16_ms"] = ms_ref
        key = f"tt{tt}" if tt else "auto"
        out[key] = res
        out[f"{key}_layer_ms"] = sum(v["ms"] for v in res.values())
        sw.close()
    out["torch_dense_layer_ms"] = sum(v["torch_matmul_bf16_ms"] for v in out["auto"].values())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
