"""Fused switch + decode on the GPU (-m gpu).

lsw_decode_token_fused runs the router and ONE launch (the fold mode of the fc
kernel) that switches every adapted matrix and computes the group GEMVs from
the freshly rounded tiles,
in decoder order with a segment barrier per (layer, group).  Checked through
the C ABI: the weights after every token are bitwise those of the separate
path (lsw_decode_token: switch launch + GEMV launches), the outputs equal its
outputs up to fp32 summation order, and the first token's outputs match the
oracle's GEMV on the oracle's merged weights; small grids make every CTA
cross many segment barriers.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests import parity as PT

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2405_17741_b200 as L
    from paper_2405_17741_b200 import harness as H


def _f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


@pytest.mark.parametrize("name,grid,tb", [("mini", None, None), ("mini", "3", None), ("mini", "1", None),
                                          ("mini-r32", None, None), ("mini-k1", "5", None), ("mini-r4k4", "2", None),
                                          ("mini-r4k4", "2", 0)])
def test_fused_token_equals_separate_path(lsw_opts, name, grid, tb):
    """tb = 0: the shared-memory fold explicitly (the fused decode is built on
    it; a ctx whose switch holds its strip in TMEM, option tc_tb = 1, refuses
    the fused decode: test_fused_refuses_tmem_strip_ctx)."""
    lsw_opts(tc_kernel="fold", tc_grid=grid, tc_tb=tb)
    cfg = synth.get_config(name)
    ctxs = []
    for _ in range(2):
        W, A, B, router = H.build_weights(cfg, "cuda")
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        ctxs.append((sw, W, A, B))
    info = ctxs[0][0].info()
    assert info["switch_kernel"] in (3, 7)
    X1 = synth.gen_x1(cfg, 5, "cuda")
    xs_d = synth.gen_xs(cfg, "cuda")
    xs = H.pack_xs(cfg, xs_d)
    outs = [dict(ys=torch.empty(info["ys_elems"], device="cuda"),
                 idx=torch.empty(cfg.top_k, dtype=torch.int32, device="cuda"),
                 gate=torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")) for _ in range(2)]
    P = {kd: _f64(ctxs[0][1][kd]) for kd in synth.KINDS}
    for t in range(4):
        (sa, Wa, Aa, Ba), (sb, Wb, _, _) = ctxs
        oa, ob = outs
        sa.decode_token(X1[t], xs, oa["ys"], oa["idx"], oa["gate"])
        n0 = sb.info()["kernel_launches"]
        sb.decode_token_fused(X1[t], xs, ob["ys"], ob["idx"], ob["gate"])
        assert sb.info()["kernel_launches"] - n0 == 2          # router + the fused launch
        torch.cuda.synchronize()
        assert sa.device_status() == 0 and sb.device_status() == 0
        assert torch.equal(oa["idx"], ob["idx"]) and torch.equal(oa["gate"], ob["gate"])
        for kd in synth.KINDS:
            assert torch.equal(Wa[kd], Wb[kd]), (t, kd)
        ya, yb = oa["ys"].cpu().numpy(), ob["ys"].cpu().numpy()
        np.testing.assert_allclose(yb, ya, rtol=1e-4, atol=1e-4 * float(np.abs(ya).max()))
        if t == 0:
            # first token: a plain merge; outputs vs the oracle's GEMV on its merged weights
            cur = (ob["idx"].cpu().tolist(), ob["gate"].cpu().double().tolist())
            scale = cfg.alpha / cfg.rank
            yo = 0
            for l in range(cfg.n_layers):
                for gi, grp in enumerate(synth.GROUPS):
                    x = _f64(xs_d[(l, gi)])
                    for kd in grp:
                        d_out = cfg.kind_shape(kd)[0]
                        Wm = O.merge(P[kd][l], _f64(Aa[kd][l]), _f64(Ba[kd][l]), cur, scale, "bf16")
                        ref = O.gemv(Wm, x)
                        assert PT.allclose_frac_fail(yb[yo:yo + d_out], ref) == 0.0, (l, kd)
                        yo += d_out


def test_fused_and_plain_tokens_alternate_on_one_ctx():
    """Plain tokens (switch launch + GEMV launches) and fused tokens alternate
    on the same W and decision slot: W stays on the oracle's stored
    trajectory and every token's outputs match the oracle's GEMV on it."""
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    info = sw.info()
    assert info["switch_kernel"] in (3, 7)
    Ws = {(kd, l): _f64(W[kd][l]) for kd in synth.KINDS for l in range(cfg.n_layers)}
    As = {(kd, l): _f64(A[kd][l]) for kd in synth.KINDS for l in range(cfg.n_layers)}
    Bs = {(kd, l): _f64(B[kd][l]) for kd in synth.KINDS for l in range(cfg.n_layers)}
    orc = O.OracleModel(_f64(router), Ws, As, Bs, cfg.top_k, cfg.alpha, cfg.rank, "bf16")
    X1 = synth.gen_x1(cfg, 4, "cuda")
    xs_d = synth.gen_xs(cfg, "cuda")
    xs = H.pack_xs(cfg, xs_d)
    ys = torch.empty(info["ys_elems"], device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    for t in range(4):
        if t % 2:
            sw.decode_token_fused(X1[t], xs, ys, idx, gate)
        else:
            sw.decode_token(X1[t], xs, ys, idx, gate)
        torch.cuda.synchronize()
        assert sw.device_status() == 0
        idx_o, g_o, _ = orc.route(_f64(X1[t]))
        assert idx.cpu().tolist() == idx_o.tolist()
        orc.merge_all_layers((idx_o.tolist(), g_o.tolist()))
        yb = ys.cpu().numpy()
        yo = 0
        for l in range(cfg.n_layers):
            for gi, grp in enumerate(synth.GROUPS):
                x = _f64(xs_d[(l, gi)])
                for kd in grp:
                    assert PT.allclose_frac_fail(_f64(W[kd][l]), orc.W[(kd, l)]) == 0.0, (t, l, kd)
                    d_out = cfg.kind_shape(kd)[0]
                    ref = O.gemv(orc.W[(kd, l)], x)
                    assert PT.allclose_frac_fail(yb[yo:yo + d_out], ref) == 0.0, (t, l, kd)
                    yo += d_out


@pytest.mark.parametrize("adapt", [None, "0"])
@pytest.mark.parametrize("name,grid", [("mini", None), ("mini", "3"), ("mini-r32", None)])
def test_fused_outputs_are_bitwise_reproducible(lsw_opts, name, grid, adapt):
    """The fc fused launch accumulates each row's per-tile contributions in
    64-bit fixed point (integer adds commute), so two runs on identical inputs
    give bitwise-identical outputs whatever order the tiles finish in
    (SURVEY §8c.5 item 5), not only bitwise-identical weights -- also under the
    adaptive split (default), which moves tiles between CTAs from pass to
    pass by measured speed (each tile's partial is converted to fixed point
    before any sum), and with the even split (adapt "0")."""
    lsw_opts(tc_kernel="fold", tc_grid=grid, fc_adapt=adapt)
    cfg = synth.get_config(name)
    X1 = synth.gen_x1(cfg, 3, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    outs = []
    for _ in range(2):
        W, A, B, router = H.build_weights(cfg, "cuda")
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        info = sw.info()
        assert info["switch_kernel"] in (3, 7)
        ys = torch.empty(info["ys_elems"], device="cuda")
        idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
        run = []
        for t in range(3):
            sw.decode_token_fused(X1[t], xs, ys, idx, gate)
            torch.cuda.synchronize()
            assert sw.device_status() == 0
            run.append((ys.clone(), {kd: W[kd].clone() for kd in synth.KINDS}))
        outs.append(run)
    for (ya, Wa), (yb, Wb) in zip(*outs):
        assert torch.equal(ya, yb)
        for kd in synth.KINDS:
            assert torch.equal(Wa[kd], Wb[kd])


@pytest.mark.parametrize("grid", [None, "3"])
def test_fused_repeated_decision_still_computes_outputs(lsw_opts, grid):
    """A token whose decision equals the merged one has an empty coefficient
    list (R12): W is unchanged, but the fused launch must still stream W and
    compute y = W x (it used to return zeros).  Checked against the
    separate path on the same ctx state, and an invalid decision (latched,
    W untouched) likewise still yields W x."""
    lsw_opts(tc_kernel="fold", tc_grid=grid)
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    info = sw.info()
    X1 = synth.gen_x1(cfg, 2, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    ya = torch.empty(info["ys_elems"], device="cuda")
    yb = torch.empty(info["ys_elems"], device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    sw.decode_token_fused(X1[0], xs, ya, idx, gate)
    torch.cuda.synchronize()
    snap = {kd: W[kd].clone() for kd in synth.KINDS}
    sw.decode_token_fused(X1[0], xs, yb, idx, gate)          # same x1 -> same decision: nothing to add
    torch.cuda.synchronize()
    assert sw.device_status() == 0
    for kd in synth.KINDS:
        assert torch.equal(W[kd], snap[kd])
    assert torch.equal(ya, yb)                              # same W, same x: bitwise (fixed-point sums)
    yc = torch.empty(info["ys_elems"], device="cuda")
    sw.decode_all_layers(xs, yc)
    torch.cuda.synchronize()
    np.testing.assert_allclose(yb.cpu().numpy(), yc.cpu().numpy(), rtol=1e-4,
                               atol=1e-4 * float(yc.abs().max()))
    assert float(yb.abs().max()) > 0
    x1 = X1[1].clone()
    x1[0] = float("nan")                                     # non-finite logits: rejected decision
    sw.decode_token_fused(x1, xs, yb, idx, gate)
    torch.cuda.synchronize()
    assert sw.device_status() == 1
    for kd in synth.KINDS:
        assert torch.equal(W[kd], snap[kd])
    assert torch.equal(ya, yb)


def test_fused_refuses_tmem_strip_ctx(lsw_opts):
    """The fused decode runs the shared-memory fold's epilogue: a ctx created
    with the TMEM-strip switch (option tc_tb = 1, mode 7) refuses it with
    LSW_E_UNSUPPORTED before enqueuing anything."""
    from paper_2405_17741_b200 import binding as L
    lsw_opts(tc_tb=1)
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    assert sw.info()["switch_kernel"] == 7
    X1 = synth.gen_x1(cfg, 1, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    ys = torch.empty(sw.info()["ys_elems"], device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    with pytest.raises(L.LswError, match="UNSUPPORTED"):
        sw.decode_token_fused(X1[0], xs, ys, idx, gate)
    assert sw.device_status() == 0
