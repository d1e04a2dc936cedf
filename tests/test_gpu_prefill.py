"""Unmerged prefill vs the oracle (-m gpu).

lsw_prefill_group evaluates Eq. 2 for T prompt tokens, each with its
own pre-gated decision (the router applied to that token's x¹): bf16 on the
tcgen05 path (LoRA-down GEMM over every expert, split K; (hi, lo) Z build; one
contraction per tile over d_in + 2 N rp), fp32 / SIMT switch on the CUDA-core
path.  Checked through the C ABI against oracle.unmerged_forward token by
token (fp64): every row at mini sizes (several 128-token tiles with a ragged
tail, rp = 16 / 32 / 64, k = 1 .. 4), sampled rows at the full widths of the
7B and 13B shapes (K = 4096 / 5120 / 11008 / 13824, split-K LoRA-down); the
result is deterministic; a merged ctx is refused.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2405_17741_b200 as L
    from paper_2405_17741_b200 import harness as H


def _f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


@pytest.mark.parametrize("name,impl,T,tt", [("toy", "simt", 5, None), ("mini", "tc", 7, None),
                                            ("mini-r64k3", "tc", 3, None), ("mini-r4k4", "tc", 33, None),
                                            ("mini", "tc", 300, None), ("mini-r32", "tc", 129, None),
                                            ("mini-k1", "tc", 130, None), ("mini-r64k4", "tc", 64, None),
                                            ("mini", "simt", 9, None), ("mini", "tc", 300, 256),
                                            ("mini-r32", "tc", 257, 256), ("mini-r4k4", "tc", 20, 256),
                                            ("mini", "tc", 512, "128/4"), ("mini", "tc", 300, "128/4"),
                                            ("mini-r32", "tc", 256, "128/2"), ("mini-r64k3", "tc", 384, "128/2"),
                                            ("mini", "tc", 1024, "256/4"), ("mini-k1", "tc", 200, "128/1"),
                                            ("mini", "tc", 512, None), ("mini-r32", "tc", 256, None),
                                            ("mini", "tc", 300, "nopair"), ("mini-r64k3", "tc", 512, "nopair"),
                                            ("mini-r64k4", "tc", 257, 128), ("mini-r4k4", "tc", 512, 256),
                                            ("mini", "tc", 300, "pair"), ("mini-r32", "tc", 512, "pair"),
                                            ("mini-r64k4", "tc", 200, "pair"), ("mini-k1", "tc", 77, "pair"),
                                            ("mini", "tc", 300, "unfused"), ("mini-r64k3", "tc", 512, "unfused"),
                                            ("mini-r4k4", "tc", 129, "unfused"), ("mini-r32", "tc", 1, "nopair"),
                                            ("mini", "tc", 300, "pair-unfused"), ("mini-r64k4", "tc", 512, "pair-unfused"),
                                            ("mini-N64", "tc", 200, None), ("mini-r48", "tc", 300, "pair"),
                                            ("mini", "tc", 300, "nosplit"), ("mini-r64k4", "tc", 257, "nosplit"),
                                            ("mini-r4k4", "tc", 64, "nosplit")])
def test_prefill_matches_oracle(lsw_opts, name, impl, T, tt):
    """The dense + LoRA-up launch runs on CTA pairs (cta_group::2, M = 256)
    for groups with a wave of 256-token tiles whose sites' row tiles pair up;
    "pair": on pairs whenever the row tiles pair up (mini: o, gate|up, down;
    not q|k|v, k being one row tile; option pf_pair=2); "nopair": single
    CTAs everywhere (pf_pair=0).  The single-CTA dense launch computes the
    LoRA-down and builds Z itself (A-bank tiles, option pf_fuse_u=1, the
    default; each bank tile's K in two halves on two CTAs when the launch is
    one wave, "nosplit": pf_bank_split=0); "unfused" / "pair-unfused": three launches (LoRA-down, Z build,
    dense + LoRA-up; pf_fuse_u=0).  tt: the token tile of the tensor-core path forced to 128 /
    256 (variant option pf_tt), or "tile/cluster": also the cluster of the dense launch forced
    (pf_cluster: W rows multicast across the token tiles of a cluster; T = 300
    with 4 pads a cluster with an all-out-of-range token tile)."""
    if tt == "nopair":                              # dense + LoRA-up on single CTAs (pf_pair=0)
        lsw_opts(pf_pair=0)
    elif tt == "pair":                              # on CTA pairs whenever the row tiles pair up (pf_pair=2)
        lsw_opts(pf_pair=2)
    elif tt == "unfused":                           # LoRA-down and Z build as launches of their own
        lsw_opts(pf_pair=0, pf_fuse_u=0)
    elif tt == "pair-unfused":
        lsw_opts(pf_pair=2, pf_fuse_u=0)
    elif tt == "nosplit":                           # fused, each A-bank tile's whole K on one CTA
        lsw_opts(pf_pair=0, pf_bank_split=0)
    elif isinstance(tt, str):
        t_, c_ = tt.split("/")
        lsw_opts(pf_tt=int(t_), pf_cluster=int(c_))
    else:
        lsw_opts(pf_tt=tt)
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl=impl)
    X1 = synth.gen_x1(cfg, T, "cuda")
    k = cfg.top_k
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gate = torch.empty(T, k, dtype=torch.float32, device="cuda")
    for t in range(T):                              # each token's own pre-gated decision (Eq. 2)
        sw.router_topk(X1[t], idx[t], gate[t])
    torch.cuda.synchronize()
    scale = cfg.alpha / cfg.rank
    g = torch.Generator(device="cpu").manual_seed(2405177410 + 99)
    for l in range(cfg.n_layers):
        for gi, grp in enumerate(synth.GROUPS):
            d_in = cfg.kind_shape(grp[0])[1]
            rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
            X = torch.randn(T, d_in, generator=g).to(W[grp[0]].dtype).cuda()
            Y = torch.full((T, rows), float("nan"), device="cuda")
            sw.prefill_group(l, gi, X, idx, gate, Y)
            torch.cuda.synchronize()
            Y2 = torch.full((T, rows), float("nan"), device="cuda")
            sw.prefill_group(l, gi, X, idx, gate, Y2)
            torch.cuda.synchronize()
            assert torch.equal(Y, Y2)               # deterministic
            Yh = Y.cpu().numpy()
            for t in range(T):
                coefs = [(int(e), scale * float(gv)) for e, gv in zip(idx[t].tolist(), gate[t].tolist())]
                o = 0
                for kd in grp:
                    d_out = cfg.kind_shape(kd)[0]
                    ref = O.unmerged_forward(_f64(W[kd][l]), _f64(A[kd][l]), _f64(B[kd][l]), coefs, _f64(X[t]))
                    np.testing.assert_allclose(Yh[t, o:o + d_out], ref, rtol=1e-4,
                                               atol=1e-4 * float(np.abs(ref).max()))
                    o += d_out
    assert sw.device_status() == 0


def test_prefill_refused_on_a_merged_ctx():
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    idx = torch.zeros(2, cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(2, cfg.top_k, dtype=torch.float32, device="cuda")
    i1 = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    g1 = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    sw.router_topk(synth.gen_x1(cfg, 1, "cuda")[0], i1, g1)
    sw.merge_all_layers(i1, g1)
    X = torch.zeros(2, cfg.d_model, dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(2, sum(cfg.kind_shape(kd)[0] for kd in synth.GROUPS[0]), device="cuda")
    with pytest.raises(L.LswError) as ei:
        sw.prefill_group(0, 0, X, idx, gate, Y)
    assert "STATE" in str(ei.value)


def _rows(d_out, seed):
    base = {0, 1, 127, 128, 129, d_out - 1}
    base |= set(np.random.default_rng(seed).choice(d_out, size=12, replace=False).tolist())
    return sorted(r for r in base if 0 <= r < d_out)


@pytest.mark.slow
@pytest.mark.parametrize("name,T", [("llama2-7b", 300), ("llama2-7b", 512), ("llama2-13b", 200)])
def test_prefill_full_width_sampled_rows(name, T):
    """One layer at the real widths: every group (K = d_model and K = d_ff),
    every token, sampled rows of every site (row sampling is exact: row i of Y
    needs row i of W and B and all of A)."""
    cfg = synth.get_config(name).with_(n_layers=1)
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    X1 = synth.gen_x1(cfg, T, "cuda")
    k = cfg.top_k
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gate = torch.empty(T, k, dtype=torch.float32, device="cuda")
    for t in range(T):
        sw.router_topk(X1[t], idx[t], gate[t])
    scale = cfg.alpha / cfg.rank
    g = torch.Generator(device="cpu").manual_seed(2405177410 + 98)
    idx_h, gate_h = idx.cpu().tolist(), gate.cpu().tolist()
    for gi, grp in enumerate(synth.GROUPS):
        d_in = cfg.kind_shape(grp[0])[1]
        rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
        X = torch.randn(T, d_in, generator=g).to(torch.bfloat16).cuda()
        Y = torch.full((T, rows), float("nan"), device="cuda")
        sw.prefill_group(0, gi, X, idx, gate, Y)
        torch.cuda.synchronize()
        Yh, Xh = Y.cpu().numpy(), _f64(X)
        o = 0
        for i, kd in enumerate(grp):
            d_out = cfg.kind_shape(kd)[0]
            rs = _rows(d_out, 31 + 7 * gi + i)
            Wr, Ar, Br = _f64(W[kd][0][rs]), _f64(A[kd][0]), _f64(B[kd][0][:, rs, :])
            for t in range(T):
                coefs = [(int(e), scale * float(gv)) for e, gv in zip(idx_h[t], gate_h[t])]
                ref = O.unmerged_forward(Wr, Ar, Br, coefs, Xh[t])
                np.testing.assert_allclose(Yh[t, o + np.array(rs)], ref, rtol=1e-4,
                                           atol=1e-4 * float(np.abs(ref).max()), err_msg=f"{kd} t={t}")
            o += d_out
        assert not np.isnan(Yh).any()
    assert sw.device_status() == 0
