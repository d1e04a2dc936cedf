"""Restore-from-pristine switch on the GPU vs the oracle (-m gpu).

lsw_restore_merge_all_layers writes W <- RNE(P + Delta(d_t)) from a pristine
copy P in one launch.  Checked through the C ABI against oracle.restore on
the same seeded inputs (allclose on every element, at most a few 1-ulp
flips), for SIMT and every mode of the tensor-core kernel; its defining property -- no
history -- bitwise: after any trajectory the result equals a fresh ctx's
restore of the same decision; and the state machine around it (restore from
`none`, fused switch and unmerge after a restore, restore without P refused).
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


def _ctx(cfg, impl):
    W, A, B, router = H.build_weights(cfg, "cuda")
    P = {kd: W[kd].clone() for kd in synth.KINDS}
    sw = H.make_switch(cfg, W, A, B, router, impl=impl)
    sw.attach_pristine(P)
    return sw, W, A, B, router, P


CASES = [("toy", "simt", None), ("mini", "tc", "fold"), ("mini", "tc", "pt"), ("mini", "tc", "bu"),
         ("mini-r4k4", "tc", None), ("mini-r64k3", "tc", None), ("mini-r64k4", "tc", None), ("mini-k1", "tc", None)]


@pytest.mark.parametrize("name,impl,kernel", CASES)
def test_restore_matches_oracle_and_has_no_history(lsw_opts, name, impl, kernel):
    lsw_opts(tc_kernel=kernel)
    cfg = synth.get_config(name)
    store = "bf16" if cfg.dtype == "bf16" else "f32"
    scale = cfg.alpha / cfg.rank
    sw, W, A, B, router, P = _ctx(cfg, impl)
    X1 = synth.gen_x1(cfg, 6, "cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    Pn = {kd: _f64(P[kd]) for kd in synth.KINDS}
    An = {kd: _f64(A[kd]) for kd in synth.KINDS}
    Bn = {kd: _f64(B[kd]) for kd in synth.KINDS}
    n0 = sw.info()["kernel_launches"]
    for t in range(5):
        sw.router_topk(X1[t], idx, gate)
        if t == 2:
            sw.merge_all_layers(idx, gate)          # a fused switch in between: restore must not care
            sw.router_topk(X1[t + 1], idx, gate)
        sw.restore_merge_all_layers(idx, gate)
        torch.cuda.synchronize()
        assert sw.device_status() == 0
        cur = (idx.cpu().tolist(), gate.cpu().double().tolist())
        for kd in synth.KINDS:
            for l in range(cfg.n_layers):
                Wo = O.restore(Pn[kd][l], An[kd][l], Bn[kd][l], cur, scale, store)
                Wg = _f64(W[kd][l])
                assert PT.allclose_frac_fail(Wg, Wo) == 0.0, (t, kd, l)
                if store == "bf16":      # one RNE from fp32 vs from fp64: rare 1-ulp flips (R14)
                    assert PT.ulp_flip_frac(Wg, Wo) <= 2e-3, (t, kd, l)
    # exactly one launch per restore (plus routers and the one fused switch)
    assert sw.info()["kernel_launches"] - n0 == 5 + 1 + 5 + 1
    # no history: a fresh ctx restoring the same decision from the same P is bitwise equal
    sw2, W2, *_ = _ctx(cfg, impl)
    sw2.restore_merge_all_layers(idx, gate)
    torch.cuda.synchronize()
    for kd in synth.KINDS:
        assert torch.equal(W[kd], W2[kd]), kd
    # and it is not a no-op of the copy: W differs from P
    assert not all(torch.equal(W[kd], P[kd]) for kd in synth.KINDS)


def test_restore_state_machine():
    cfg = synth.get_config("mini")
    scale = cfg.alpha / cfg.rank
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    X1 = synth.gen_x1(cfg, 3, "cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    sw.router_topk(X1[0], idx, gate)
    with pytest.raises(L.LswError) as ei:
        sw.restore_merge_all_layers(idx, gate)            # no pristine copy yet
    assert "STATE" in str(ei.value)
    P = {kd: W[kd].clone() for kd in synth.KINDS}
    sw.attach_pristine(P)
    assert sw.info()["merged"] == 0
    sw.restore_merge_all_layers(idx, gate)                # from state none
    assert sw.info()["merged"] == 1
    d1 = (idx.cpu().tolist(), gate.cpu().double().tolist())
    W1 = {kd: _f64(W[kd]) for kd in synth.KINDS}
    # fused switch after a restore removes d1's delta (the decision was recorded)
    sw.router_topk(X1[1], idx, gate)
    sw.merge_all_layers(idx, gate)
    torch.cuda.synchronize()
    d2 = (idx.cpu().tolist(), gate.cpu().double().tolist())
    for kd in synth.KINDS:
        for l in range(cfg.n_layers):
            Wo = O.switch(W1[kd][l], _f64(A[kd][l]), _f64(B[kd][l]), d1, d2, scale, "bf16")
            assert PT.allclose_frac_fail(_f64(W[kd][l]), Wo) == 0.0
    # unmerge returns to (approximately) the pristine weights
    sw.unmerge_all_layers()
    torch.cuda.synchronize()
    for kd in synth.KINDS:
        assert PT.allclose_frac_fail(_f64(W[kd]), _f64(P[kd])) == 0.0
    assert sw.device_status() == 0


@pytest.mark.parametrize("name,kernel,grid", [("mini", "fold", None), ("mini", "pt", "3"), ("mini", "fold", "3"),
                                                  ("mini-r4k4", None, None), ("mini-r64k4", "bu", "2")])
def test_per_matrix_merge_ablation_is_bitwise_the_single_launch(lsw_opts, name, kernel, grid):
    """SURVEY 8f #4 (launch-count ablation): the merge as one launch per matrix
    (7 x L launches of the same kernel over that matrix's tiles) gives bitwise
    the same weights as the single all-layer launch, and records the decision
    (a fused switch afterwards is correct)."""
    lsw_opts(tc_kernel=kernel, tc_grid=grid)
    cfg = synth.get_config(name)
    outs = []
    for mode in ("single", "per_matrix"):
        W, A, B, router = H.build_weights(cfg, "cuda")
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        X1 = synth.gen_x1(cfg, 2, "cuda")
        idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
        sw.router_topk(X1[0], idx, gate)
        n0 = sw.info()["kernel_launches"]
        if mode == "single":
            sw.merge_all_layers(idx, gate)
            assert sw.info()["kernel_launches"] - n0 == 1
        else:
            sw.debug_merge_per_matrix(idx, gate)
            assert sw.info()["kernel_launches"] - n0 == 7 * cfg.n_layers
            with pytest.raises(L.LswError):
                sw.debug_merge_per_matrix(idx, gate)        # merged: refused
        merged = {kd: W[kd].clone() for kd in synth.KINDS}
        sw.router_topk(X1[1], idx, gate)
        sw.merge_all_layers(idx, gate)                        # fused switch from the recorded decision
        torch.cuda.synchronize()
        assert sw.device_status() == 0
        outs.append((merged, {kd: W[kd].clone() for kd in synth.KINDS}))
    for kd in synth.KINDS:
        assert torch.equal(outs[0][0][kd], outs[1][0][kd]), kd
        assert torch.equal(outs[0][1][kd], outs[1][1][kd]), kd
