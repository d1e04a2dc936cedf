"""Tensor-parallel shards on ONE GPU (-m gpu).

SURVEY §8e: merge / unmerge / switch are local to each shard; the decode GEMV
of a row-parallel kind (o, down) needs a sum over ranks.  gpurun gives one GPU
and NCCL cannot place two ranks on one device, so this test builds the rank-0
and rank-1 shards of the same model side by side in one process, each behind
its own ctx over the LOCAL shapes (tp_size=1 view: exactly the kernels a TP
rank runs; only the NCCL all-reduce is left out), and checks through the C ABI:
(i) identical router decisions on both ranks, (ii) each shard's switched W is
the matching slice of the un-sharded result -- bitwise, the per-element
contraction does not depend on the tiling -- (iii) column-parallel GEMV outputs
are exact slices and row-parallel partial outputs sum (torch, standing in for
the all-reduce) to the full output within fp32 ordering tolerance.  A
tp_size=2 ctx without a communicator must refuse a row-parallel decode before
enqueuing anything.
"""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2405_17741_b200 as L
    from paper_2405_17741_b200 import harness as H


@pytest.mark.parametrize("name,impl,size", [("mini", "tc", 2), ("mini", "simt", 2), ("mini-r32", "tc", 2),
                                            ("mini", "tc", 4), ("mini-r32", "tc", 8), ("mini-r64k3", "tc", 4)])
def test_tp_shards_match_full_model(name, impl, size):
    """size 4 / 8: ragged shards (d_ff 704 -> 176 / 88 columns of down, d_model
    256 -> 32 columns of o: 3-D W boxes instead of the row-major 4-D view,
    partial tiles) through the same kernels; r = 64, k = 3: the per-term mode."""
    cfg = synth.get_config(name)
    full = H.build_weights(cfg, "cuda")
    sw_full = H.make_switch(cfg, *full, impl=impl)
    shards = [H.build_weights(cfg, "cuda", r, size) for r in range(size)]
    sws = [H.make_switch(cfg, *shards[r], impl=impl) for r in range(size)]     # local-shape view
    X1 = synth.gen_x1(cfg, 4, "cuda")
    xs = synth.gen_xs(cfg, "cuda")
    k = cfg.top_k
    idx = [torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(size + 1)]
    gate = [torch.empty(k, dtype=torch.float32, device="cuda") for _ in range(size + 1)]
    for t in range(4):
        sw_full.router_topk(X1[t], idx[size], gate[size])
        sw_full.merge_all_layers(idx[size], gate[size])
        for r in range(size):
            sws[r].router_topk(X1[t], idx[r], gate[r])
            sws[r].merge_all_layers(idx[r], gate[r])
        torch.cuda.synchronize()
        for r in range(size):
            assert torch.equal(idx[r], idx[size]) and torch.equal(gate[r], gate[size])
    for r in range(size):
        for kd in synth.KINDS:
            ref = synth.shard_W(cfg, kd, full[0][kd], r, size)
            assert torch.equal(shards[r][0][kd], ref), (name, impl, kd, r)
    for l in range(cfg.n_layers):
        for gi, grp in enumerate(synth.GROUPS):
            for kd in grp:
                y_full = torch.empty(cfg.kind_shape(kd)[0], dtype=torch.float32, device="cuda")
                sw_full.decode_linear(l, kd, xs[(l, gi)], y_full)
                parts = []
                for r in range(size):
                    y = torch.empty(cfg.local_shape(kd, r, size)[0], dtype=torch.float32, device="cuda")
                    x = synth.shard_x(cfg, gi, xs[(l, gi)], r, size).contiguous()
                    sws[r].decode_linear(l, kd, x, y)
                    parts.append(y)
                torch.cuda.synchronize()
                if kd in synth.ROW_PARALLEL:
                    torch.testing.assert_close(sum(parts[1:], parts[0]), y_full, rtol=1e-5, atol=1e-5)
                else:
                    assert torch.equal(torch.cat(parts), y_full)
    for s in sws + [sw_full]:
        assert s.device_status() == 0


def test_tp_ctx_without_communicator_refuses_row_parallel_decode():
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda", 0, 2)
    sw = H.make_switch(cfg, W, A, B, router, impl="tc", tp_rank=0, tp_size=2)
    x = synth.shard_x(cfg, 1, synth.gen_xs(cfg, "cuda")[(0, 1)], 0, 2).contiguous()
    y = torch.full((cfg.kind_shape("o")[0],), 7.0, device="cuda")
    with pytest.raises(L.LswError) as ei:
        sw.decode_linear(0, "o", x, y)
    assert "NCCL" in str(ei.value)
    torch.cuda.synchronize()
    assert torch.all(y == 7.0)                      # nothing was enqueued
    launches = sw.info()["kernel_launches"]
    assert launches == 0
    # column-parallel kinds need no communicator
    yq = torch.empty(cfg.local_shape("q", 0, 2)[0], device="cuda")
    sw.decode_linear(0, "q", synth.gen_xs(cfg, "cuda")[(0, 0)], yq)
    assert sw.info()["kernel_launches"] == 1


def _by_site(cfg, grp, parts, size):
    """Column-parallel group outputs of the ranks [q_r | k_r | v_r] -> [q | k | v]."""
    out = []
    for i, kd in enumerate(grp):
        for r in range(size):
            off = sum(cfg.local_shape(k2, r, size)[0] for k2 in grp[:i])
            n = cfg.local_shape(kd, r, size)[0]
            out.append(parts[r][..., off:off + n])
    return torch.cat(out, dim=-1)


@pytest.mark.parametrize("name,size", [("mini", 2), ("mini-r32", 4)])
def test_tp_shards_unmerged_decode_and_prefill(name, size):
    """Unmerged decode and prefill (Eq. 2) per TP shard through the C ABI,
    local-shape view as above: column-parallel groups' rows are the full
    model's rows (bitwise for the decode), row-parallel partials sum (torch,
    standing in for the all-reduce the library issues under a communicator)
    to the full output -- Eq. 2 is linear in the d_in shards of W and A."""
    cfg = synth.get_config(name)
    full = H.build_weights(cfg, "cuda")
    sw_full = H.make_switch(cfg, *full, impl="tc")
    shards = [H.build_weights(cfg, "cuda", r, size) for r in range(size)]
    sws = [H.make_switch(cfg, *shards[r], impl="tc") for r in range(size)]
    T = 33
    X1 = synth.gen_x1(cfg, T, "cuda")
    xs = synth.gen_xs(cfg, "cuda")
    k = cfg.top_k
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gate = torch.empty(T, k, dtype=torch.float32, device="cuda")
    for t in range(T):
        sw_full.router_topk(X1[t], idx[t], gate[t])
    g = torch.Generator(device="cpu").manual_seed(2405177410 + 77)
    for l in range(cfg.n_layers):
        for gi, grp in enumerate(synth.GROUPS):
            rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
            row_par = grp[0] in synth.ROW_PARALLEL
            # decode, token 0's decision
            y_full = torch.empty(rows, device="cuda")
            sw_full.decode_group_unmerged(l, gi, xs[(l, gi)], y_full, idx[0], gate[0])
            parts = []
            for r in range(size):
                rl = sum(cfg.local_shape(kd, r, size)[0] for kd in grp)
                y = torch.empty(rl, device="cuda")
                x = synth.shard_x(cfg, gi, xs[(l, gi)], r, size).contiguous()
                sws[r].decode_group_unmerged(l, gi, x, y, idx[0], gate[0])
                parts.append(y)
            # prefill, every token its own decision
            d_in = cfg.kind_shape(grp[0])[1]
            X = torch.randn(T, d_in, generator=g).to(full[0][grp[0]].dtype).cuda()
            Y_full = torch.empty(T, rows, device="cuda")
            sw_full.prefill_group(l, gi, X, idx, gate, Y_full)
            Yparts = []
            for r in range(size):
                rl = sum(cfg.local_shape(kd, r, size)[0] for kd in grp)
                Y = torch.empty(T, rl, device="cuda")
                Xr = torch.stack([synth.shard_x(cfg, gi, X[t], r, size) for t in range(T)]).contiguous()
                sws[r].prefill_group(l, gi, Xr, idx, gate, Y)
                Yparts.append(Y)
            torch.cuda.synchronize()
            if row_par:
                torch.testing.assert_close(sum(parts[1:], parts[0]), y_full, rtol=1e-5, atol=1e-5)
                torch.testing.assert_close(sum(Yparts[1:], Yparts[0]), Y_full, rtol=1e-5, atol=1e-4)
            else:
                assert torch.equal(_by_site(cfg, grp, parts, size), y_full), (name, l, gi)
                torch.testing.assert_close(_by_site(cfg, grp, Yparts, size), Y_full, rtol=1e-5, atol=1e-5)
    for s in sws + [sw_full]:
        assert s.device_status() == 0


def test_tp_ctx_without_communicator_refuses_row_parallel_unmerged():
    """tp_size = 2 and no communicator: the row-parallel unmerged decode and
    prefill are refused before anything is enqueued; column-parallel run."""
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda", 0, 2)
    sw = H.make_switch(cfg, W, A, B, router, impl="tc", tp_rank=0, tp_size=2)
    idx = torch.tensor(list(range(cfg.top_k)), dtype=torch.int32, device="cuda")
    gate = torch.full((cfg.top_k,), 1.0 / cfg.top_k, device="cuda")
    x = synth.shard_x(cfg, 1, synth.gen_xs(cfg, "cuda")[(0, 1)], 0, 2).contiguous()
    y = torch.full((cfg.local_shape("o", 0, 2)[0],), 7.0, device="cuda")
    with pytest.raises(L.LswError) as ei:
        sw.decode_group_unmerged(0, 1, x, y, idx, gate)
    assert "NCCL" in str(ei.value)
    X = torch.zeros(3, x.numel(), dtype=x.dtype, device="cuda")
    Y = torch.zeros(3, y.numel(), device="cuda")
    with pytest.raises(L.LswError) as ei:
        sw.prefill_group(0, 1, X, idx.repeat(3, 1), gate.repeat(3, 1), Y)
    assert "NCCL" in str(ei.value)
    torch.cuda.synchronize()
    assert torch.all(y == 7.0) and sw.info()["kernel_launches"] == 0
    rows = sum(cfg.local_shape(kd, 0, 2)[0] for kd in synth.GROUPS[0])
    yq = torch.empty(rows, device="cuda")
    sw.decode_group_unmerged(0, 0, synth.gen_xs(cfg, "cuda")[(0, 0)], yq, idx, gate)
    assert sw.info()["kernel_launches"] == 1
