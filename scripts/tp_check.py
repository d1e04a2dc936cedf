"""Tensor-parallel decode through the C ABI on N GPUs (torchrun worker; SURVEY
§8e, row a-6).  Each rank builds its shard of the same seeded model (column
split: q, k, v, gate, up; row split: o, down), attaches an NCCL communicator
with lsw_attach_nccl (unique id broadcast over torch.distributed), runs T
tokens of lsw_decode_token (router -> one switch launch -> GEMVs with the
fp32 all-reduce of o / down), and checks against the oracle on the FULL
weights: identical decisions on every rank, each W shard within the parity
tolerance of the oracle's slice, column-parallel outputs equal to the oracle's
rows, row-parallel outputs (after the all-reduce) equal to the oracle's full
output; then the unmerged decode (lsw_decode_all_layers_unmerged, o / down
partials all-reduced) against the oracle's Eq. 2.  Rank 0 prints one JSON
line; exit code 0 iff every rank passed.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 scripts/tp_check.py [--config mini] [--tokens 3]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402
from paper_2405_17741_b200.binding import LoraSwitch, nccl_version  # noqa: E402
from tests import parity as PT  # noqa: E402


def f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mini")
    ap.add_argument("--tokens", type=int, default=3)
    ap.add_argument("--impl", default="auto")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.get_config(a.config)
    store = "bf16" if cfg.dtype == "bf16" else "f32"
    W, A, B, router = H.build_weights(cfg, "cuda", rank, world)
    sw = H.make_switch(cfg, W, A, B, router, impl=a.impl, tp_rank=rank, tp_size=world)
    uid = [LoraSwitch.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    sw.attach_nccl(uid[0])
    info = sw.info()
    # oracle on the full (un-sharded) weights, sliced per rank afterwards
    Ws, As, Bs = {}, {}, {}
    for kd in synth.KINDS:
        for l in range(cfg.n_layers):
            Ws[(kd, l)] = f64(synth.gen_W(cfg, kd, l))
            As[(kd, l)] = f64(synth.gen_A(cfg, kd, l))
            Bs[(kd, l)] = f64(synth.gen_B(cfg, kd, l))
    orc = O.OracleModel(f64(synth.gen_router(cfg)), Ws, As, Bs, cfg.top_k, cfg.alpha, cfg.rank, store)
    X1 = synth.gen_x1(cfg, a.tokens, "cuda")
    xs_full = synth.gen_xs(cfg, "cuda")
    xs = H.pack_xs(cfg, xs_full, rank, world)
    ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    layout, _ = H.ys_layout(cfg, rank, world)
    errs = []
    worst = {"w_div": 0.0, "y_fail": 0.0}
    for t in range(a.tokens):
        sw.decode_token(X1[t], xs, ys, idx, gate)
        torch.cuda.synchronize()
        io, go, _ = orc.route(f64(X1[t]))
        orc.merge_all_layers((io.tolist(), go.tolist()))
        if idx.cpu().tolist() != io.tolist():
            errs.append(f"t{t}: idx {idx.cpu().tolist()} != oracle {io.tolist()}")
        dec = [None] * world
        dist.all_gather_object(dec, (idx.cpu().tolist(), gate.cpu().tolist()))
        if any(d != dec[0] for d in dec):
            errs.append(f"t{t}: decisions differ across ranks")
        yh = ys.cpu().numpy()
        for (l, kd, off, n) in layout:
            gi = next(i for i, g in enumerate(synth.GROUPS) if kd in g)
            x = f64(xs_full[(l, gi)])
            y_full = O.gemv(orc.W[(kd, l)], x)
            if kd in synth.ROW_PARALLEL:
                ref = y_full                          # all-reduced over the ranks
            else:
                lo, hi = synth.shard_range(cfg.kind_shape(kd)[0], rank, world)
                ref = y_full[lo:hi]
            fail = PT.allclose_frac_fail(yh[off:off + n], ref)
            worst["y_fail"] = max(worst["y_fail"], fail)
            if fail:
                errs.append(f"t{t} y {kd}[{l}]: {fail:.3e} outside allclose")
        for kd in synth.KINDS:
            for l in range(cfg.n_layers):
                ref = synth.shard_W(cfg, kd, torch.from_numpy(orc.W[(kd, l)]), rank, world).numpy()
                Wg = f64(W[kd][l])
                div = PT.divergence(Wg, ref)
                worst["w_div"] = max(worst["w_div"], div)
                if PT.allclose_frac_fail(Wg, ref) or div > PT.DIVERGENCE_TOL:
                    errs.append(f"t{t} W {kd}[{l}] shard {rank}: div {div:.3e}")
    sw.unmerge_all_layers()
    orc.unmerge_all_layers()
    # the unmerged decode (Eq. 2 on the unmerged weights): column-parallel rows
    # complete per rank, row-parallel partials all-reduced by the library
    sw.router_topk(X1[0], idx, gate)
    sw.decode_all_layers_unmerged(xs, ys, idx, gate)
    torch.cuda.synchronize()
    io, go, _ = orc.route(f64(X1[0]))
    coefs = [(int(e), cfg.alpha / cfg.rank * float(gv)) for e, gv in zip(io.tolist(), go.tolist())]
    yh = ys.cpu().numpy()
    worst["y_unmerged_fail"] = 0.0
    for (l, kd, off, n) in layout:
        gi = next(i for i, g in enumerate(synth.GROUPS) if kd in g)
        y_full = O.unmerged_forward(orc.W[(kd, l)], As[(kd, l)], Bs[(kd, l)], coefs, f64(xs_full[(l, gi)]))
        if kd in synth.ROW_PARALLEL:
            ref = y_full
        else:
            lo, hi = synth.shard_range(cfg.kind_shape(kd)[0], rank, world)
            ref = y_full[lo:hi]
        fail = PT.allclose_frac_fail(yh[off:off + n], ref)
        worst["y_unmerged_fail"] = max(worst["y_unmerged_fail"], fail)
        if fail:
            errs.append(f"unmerged y {kd}[{l}]: {fail:.3e} outside allclose")
    st = sw.device_status()
    if st:
        errs.append(f"device status {st}")
    v, path = nccl_version()
    res = {"rank": rank, "errors": errs[:20], "worst": worst, "nccl": v, "nccl_path": path,
           "launches": sw.info()["kernel_launches"]}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    ok = all(not r["errors"] for r in allres)
    if rank == 0:
        print(json.dumps({"ok": ok, "world": world, "config": cfg.name, "tokens": a.tokens, "ranks": allres}))
    sw.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
