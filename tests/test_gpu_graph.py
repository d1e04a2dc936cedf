"""Whole decode tokens captured in a CUDA graph (-m gpu).

include/lsw.h promises that hot calls only enqueue and that decisions never
return to the host, so a token -- lsw_decode_token: router -> one switch
launch -> the group GEMVs (PDL-chained) -- is graph-capturable; the switch
kernel keeps the merged decision in device state, so replaying the SAME graph
for a new token (its x^1 copied into the captured input buffer) performs the
Eq. 10 switch from whatever the previous replay merged.  Checked against the
same token sequence run eagerly on a second ctx over copies of the same
weights: W, outputs and decisions bitwise equal after every token, for the
tensor-core switch (fold and per-term modes) and the SIMT switch; the fused
switch + decode likewise.
"""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2405_17741_b200 import harness as H


def _pair(cfg, impl):
    out = []
    for _ in range(2):
        W, A, B, router = H.build_weights(cfg, "cuda")
        out.append((W, H.make_switch(cfg, W, A, B, router, impl=impl)))
    return out


@pytest.mark.parametrize("name,impl,fused", [("mini", "tc", False), ("mini-r64k3", "tc", False),
                                             ("toy", "simt", False), ("mini", "tc", True)])
def test_token_graph_replay_equals_eager(name, impl, fused):
    cfg = synth.get_config(name)
    (We, swe), (Wg, swg) = _pair(cfg, impl)
    X1 = synth.gen_x1(cfg, 6, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    n_ys = swe.info()["ys_elems"]
    k = cfg.top_k
    ys_e, ys_g = torch.empty(n_ys, device="cuda"), torch.empty(n_ys, device="cuda")
    idx_e, idx_g = (torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(2))
    g_e, g_g = (torch.empty(k, dtype=torch.float32, device="cuda") for _ in range(2))
    x1_static = torch.empty_like(X1[0])
    token = swg.decode_token_fused if fused else swg.decode_token
    token_e = swe.decode_token_fused if fused else swe.decode_token
    # token 0 eagerly on both ctxs (plain merge; the fused path builds its table)
    token_e(X1[0], xs, ys_e, idx_e, g_e)
    x1_static.copy_(X1[0])
    token(x1_static, xs, ys_g, idx_g, g_g)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        token(x1_static, xs, ys_g, idx_g, g_g, s)
    for t in range(1, 6):
        x1_static.copy_(X1[t])
        graph.replay()
        token_e(X1[t], xs, ys_e, idx_e, g_e)
        torch.cuda.synchronize()
        assert torch.equal(idx_g, idx_e) and torch.equal(g_g, g_e), t
        assert torch.equal(ys_g, ys_e), t
        for kd in synth.KINDS:
            assert torch.equal(Wg[kd], We[kd]), (t, kd)
    assert swg.device_status() == 0 and swe.device_status() == 0


@pytest.mark.parametrize("name,T", [("mini", 300), ("mini-r4k4", 129), ("mini-r64k3", 512)])
def test_prefill_graph_replay(lsw_opts, name, T):
    """lsw_prefill_group captured in a CUDA graph, after one eager call built
    the plan and the scratch: under capture the dense launch does not fold in
    the LoRA-down (the fused launch's completion-count target is fixed per
    launch), so the captured layer -- all four groups -- replays the
    three-launch path: bitwise equal, for new inputs copied into the captured
    buffers, to an eager ctx whose plan has the fusion off (pf_fuse_u=0)."""
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    swg = H.make_switch(cfg, W, A, B, router, impl="tc")           # default options: fused when eager
    k = cfg.top_k
    g = torch.Generator(device="cpu").manual_seed(2405177410 + 97)
    idx = torch.stack([torch.randperm(cfg.n_experts, generator=g)[:k] for _ in range(T)]).to(torch.int32).cuda()
    gate = torch.softmax(torch.randn(T, k, generator=g), dim=1).cuda()
    Xs, Ys_g, Ys_e = [], [], []
    for grp in synth.GROUPS:
        d_in = cfg.kind_shape(grp[0])[1]
        rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
        Xs.append(torch.empty(T, d_in, dtype=W[grp[0]].dtype, device="cuda"))
        Ys_g.append(torch.empty(T, rows, device="cuda"))
        Ys_e.append(torch.empty(T, rows, device="cuda"))

    def fill():
        for X in Xs:
            X.copy_(torch.randn(X.shape, generator=g).to(X.dtype))

    fill()
    for gi in range(len(synth.GROUPS)):                          # eager: plan + scratch
        swg.prefill_group(0, gi, Xs[gi], idx, gate, Ys_g[gi])
    torch.cuda.synchronize()
    lsw_opts(pf_fuse_u=0)
    swe = H.make_switch(cfg, W, A, B, router, impl="tc")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for gi in range(len(synth.GROUPS)):
            swg.prefill_group(0, gi, Xs[gi], idx, gate, Ys_g[gi], s)
    for rep in range(3):
        fill()
        graph.replay()
        for gi in range(len(synth.GROUPS)):
            swe.prefill_group(0, gi, Xs[gi], idx, gate, Ys_e[gi])
        torch.cuda.synchronize()
        for gi in range(len(synth.GROUPS)):
            assert torch.equal(Ys_g[gi], Ys_e[gi]), (rep, gi)
    assert swg.device_status() == 0 and swe.device_status() == 0
