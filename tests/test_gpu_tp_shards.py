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
