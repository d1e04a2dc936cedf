"""Tensor-parallel host logic on CPU (gloo, world_size 2) -- -m "not gpu".

SURVEY §8e: column-parallel kinds (q,k,v,gate,up) shard W/B rows and keep A
replicated; row-parallel kinds (o,down) shard W/A columns and keep B
replicated.  Merge/unmerge/switch are local per shard; the decode GEMV of a
row-parallel kind needs one sum-allreduce of the partial outputs.  Here each
rank runs the oracle on its shard (built by synth.shard_*), and the test
checks (i) each shard equals the slice of the full result bitwise, (ii) the
router decision is identical on every rank, (iii) gathered / allreduced GEMV
outputs equal the full GEMV, (iv) the unmerged forward (Eq. 2, the unmerged
decode / prefill) on the pristine shards gathers / all-reduces to the full one.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS["toy"]
        scale = cfg.alpha / cfg.rank
        Wg = synth.to_f64_numpy(synth.gen_router(cfg))
        X1 = synth.to_f64_numpy(synth.gen_x1(cfg, 3))
        xs = synth.gen_xs(cfg)
        ok = True
        decisions = []
        for t in range(3):
            idx, g, _ = O.router(Wg, X1[t], cfg.top_k)
            decisions.append((idx.tolist(), g.tolist()))
        # (ii) identical decisions on every rank
        gathered = [None] * world
        dist.all_gather_object(gathered, decisions)
        ok &= all(d == decisions for d in gathered)
        layer = 1
        for gi, grp in enumerate(synth.GROUPS):
            x_full = synth.to_f64_numpy(xs[(layer, gi)])
            x_loc = synth.to_f64_numpy(synth.shard_x(cfg, gi, xs[(layer, gi)], rank, world))
            for kd in grp:
                Wf = synth.gen_W(cfg, kd, layer)
                Af = synth.gen_A(cfg, kd, layer)
                Bf = synth.gen_B(cfg, kd, layer)
                Wl = synth.to_f64_numpy(synth.shard_W(cfg, kd, Wf, rank, world))
                Al = synth.to_f64_numpy(synth.shard_A(cfg, kd, Af, rank, world))
                Bl = synth.to_f64_numpy(synth.shard_B(cfg, kd, Bf, rank, world))
                W_full = synth.to_f64_numpy(Wf)
                A_full = synth.to_f64_numpy(Af)
                B_full = synth.to_f64_numpy(Bf)
                prev = None
                for t in range(3):
                    Wl = O.switch(Wl, Al, Bl, prev, decisions[t], scale, "f32")
                    W_full = O.switch(W_full, A_full, B_full, prev, decisions[t], scale, "f32")
                    prev = decisions[t]
                # (i) shard == slice of the full result (bitwise)
                ref = synth.shard_W(cfg, kd, torch.from_numpy(W_full), rank, world).numpy()
                ok &= bool(np.array_equal(Wl, ref))
                # (iii) decode GEMV: allreduce for row-parallel, gather for column-parallel
                y_loc = torch.from_numpy(O.gemv(Wl, x_loc))
                y_full = O.gemv(W_full, x_full)
                if kd in synth.ROW_PARALLEL:
                    dist.all_reduce(y_loc)
                    ok &= bool(np.allclose(y_loc.numpy(), y_full, rtol=1e-12, atol=1e-12))
                else:
                    parts = [torch.zeros(cfg.local_shape(kd, r_, world)[0], dtype=torch.float64)
                             for r_ in range(world)]
                    dist.all_gather(parts, y_loc)
                    ok &= bool(np.array_equal(torch.cat(parts).numpy(), y_full))
                # (iv) unmerged forward (Eq. 2) on the pristine shards: the row-parallel
                # partials W_s x_s + sum_j c_j B_j (A_j,s x_s) all-reduce to the full
                # result (linear in the d_in shards: no all-reduce of A x needed)
                coefs = [(int(e), scale * float(gv)) for e, gv in zip(*decisions[2])]
                P_loc = synth.to_f64_numpy(synth.shard_W(cfg, kd, Wf, rank, world))
                u_loc = torch.from_numpy(O.unmerged_forward(P_loc, Al, Bl, coefs, x_loc))
                u_full = O.unmerged_forward(synth.to_f64_numpy(Wf), synth.to_f64_numpy(Af),
                                            synth.to_f64_numpy(Bf), coefs, x_full)
                if kd in synth.ROW_PARALLEL:
                    dist.all_reduce(u_loc)
                    ok &= bool(np.allclose(u_loc.numpy(), u_full, rtol=1e-12, atol=1e-12))
                else:
                    parts = [torch.zeros(cfg.local_shape(kd, r_, world)[0], dtype=torch.float64)
                             for r_ in range(world)]
                    dist.all_gather(parts, u_loc)
                    ok &= bool(np.allclose(torch.cat(parts).numpy(), u_full, rtol=1e-12, atol=1e-12))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_tp2_oracle_shards_match_full_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


def test_shard_range_covers_exactly():
    for n in (64, 128, 1024, 2752, 11008, 13824, 13):
        for size in (1, 2, 3, 4, 8):
            spans = [synth.shard_range(n, r, size) for r in range(size)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(size - 1))
