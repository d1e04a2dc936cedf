"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of liblsw on mini shapes through the C ABI --
router, SIMT switch (fp32 toy), the tensor-core fc switch in its fold,
per-term and B-per-unit modes (tiny grids: every ring wraps), restore, the
fused switch + decode, the bulk GEMV (merged and unmerged), the LDG GEMV, the
prefill kernels.  Exits non-zero if a device error is latched.

  compute-sanitizer --tool memcheck python scripts/sanitize_driver.py [--quick]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def run(name, impl="auto", opts=None, tokens=3, fused=False, unmerged=False, restore=False, prefill=False):
    with binding.options(**(opts or {})):
        cfg = synth.get_config(name)
        W, A, B, router = H.build_weights(cfg, "cuda")
        Pc = {k: v.clone() for k, v in W.items()}
        sw = H.make_switch(cfg, W, A, B, router, impl=impl)
    info = sw.info()
    X1 = synth.gen_x1(cfg, tokens, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    if unmerged:
        sw.router_topk(X1[0], idx, gate)
        sw.decode_all_layers_unmerged(xs, ys, idx, gate)
    if prefill:
        T = 5
        X = torch.randn(T, cfg.d_model, device="cuda").to(cfg.torch_dtype)
        pidx = torch.stack([torch.randperm(cfg.n_experts, device="cuda")[:cfg.top_k] for _ in range(T)]).int()
        pg = torch.full((T, cfg.top_k), 1.0 / cfg.top_k, device="cuda")
        rows = sum(cfg.kind_shape(k)[0] for k in synth.GROUPS[0])
        Y = torch.empty(T, rows, device="cuda")
        sw.prefill_group(0, 0, X, pidx, pg, Y)
    for t in range(tokens):
        if fused:
            sw.decode_token_fused(X1[t], xs, ys, idx, gate)
        else:
            sw.decode_token(X1[t], xs, ys, idx, gate)
    if restore:
        sw.attach_pristine(Pc)
        sw.restore_merge_all_layers(idx, gate)
    sw.unmerge_all_layers()
    st = sw.device_status()
    sw.close()
    print(f"{name} {impl} {opts or ''} fused={fused} unmerged={unmerged}: status {st}", flush=True)
    return st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    bad = 0
    bad |= run("toy", "simt", unmerged=False)
    bad |= run("mini", "tc", {"tc_grid": 3}, unmerged=True, restore=True, prefill=True)
    bad |= run("mini", "tc", {"tc_grid": 2}, fused=True)
    bad |= run("mini-r32", "tc", {"tc_grid": 2, "gemv_grid": 3})
    if not a.quick:
        bad |= run("mini-r64k3", "tc", {"tc_grid": 2})                       # per-term
        bad |= run("mini-r64k4", "tc", {"tc_grid": 2})                       # B per unit
        bad |= run("mini", "tc", {"gemv": "ldg"})
        bad |= run("mini-r4k4", "tc", {"tc_grid": 1, "fc_stages": 3, "fc_astages": 2, "fc_bbufs": 1})
        bad |= run("mini", "simt", unmerged=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
