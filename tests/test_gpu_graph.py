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
