"""Unmerged decode (Eq. 2 at P:228 without merging) vs the oracle (-m gpu).

lsw_decode_group_unmerged computes y = W x + sum_j (alpha/r) g_j B_j (A_j x) on
the pristine weights in one launch per group (LoRA-down products dealt over
the grid and published through a device counter, LoRA-up added at the end of
each CTA's stream).  Checked through the C ABI
against oracle.unmerged_forward on the same seeded inputs (fp64), for bf16 and
fp32 storage, k*r below and above one warp (32), and k = 1..4; the whole-layer
call equals the per-group calls bitwise; the merged path (Eq. 3 on the merged
weights) agrees within the storage rounding; a merged ctx is refused.
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


@pytest.mark.parametrize("name,impl,grid", [("toy", "simt", None), ("mini", "tc", None), ("mini-r32", "tc", None),
                                            ("mini-r64k3", "tc", None), ("mini-r4k4", "tc", None),
                                            ("mini-k1", "tc", None), ("mini", "tc", "3"), ("mini-r64k3", "tc", "2")])
def test_unmerged_decode_matches_oracle(lsw_opts, name, impl, grid):
    """grid: a GEMV grid of a few CTAs, so each CTA computes many LoRA-down
    products over several warps and the device counters are reset and reused
    across many launches."""
    lsw_opts(gemv_grid=grid)
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl=impl)
    info = sw.info()
    X1 = synth.gen_x1(cfg, 3, "cuda")
    xs = synth.gen_xs(cfg, "cuda")
    xs_p = H.pack_xs(cfg, xs)
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    scale = cfg.alpha / cfg.rank
    for t in range(2):
        sw.router_topk(X1[t], idx, gate)
        coefs = [(int(e), scale * float(g)) for e, g in zip(idx.cpu().tolist(), gate.cpu().tolist())]
        ys_groups = torch.full((info["ys_elems"],), float("nan"), device="cuda")
        yo = 0
        for l in range(cfg.n_layers):
            for gi, grp in enumerate(synth.GROUPS):
                n_out = sum(cfg.kind_shape(kd)[0] for kd in grp)
                y = ys_groups[yo:yo + n_out]
                sw.decode_group_unmerged(l, gi, xs[(l, gi)], y, idx, gate)
                torch.cuda.synchronize()
                x = _f64(xs[(l, gi)])
                o = 0
                for kd in grp:
                    d_out = cfg.kind_shape(kd)[0]
                    ref = O.unmerged_forward(_f64(W[kd][l]), _f64(A[kd][l]), _f64(B[kd][l]), coefs, x)
                    got = y[o:o + d_out].cpu().numpy()
                    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-4 * float(np.abs(ref).max()))
                    o += d_out
                yo += n_out
        # whole-layer call: the same launches, bitwise
        ys_all = torch.full((info["ys_elems"],), float("nan"), device="cuda")
        sw.decode_all_layers_unmerged(xs_p, ys_all, idx, gate)
        torch.cuda.synchronize()
        assert torch.equal(ys_all, ys_groups)
    assert sw.device_status() == 0
    # Eq. 3 on the merged weights agrees with Eq. 2 within the storage rounding
    sw.merge_all_layers(idx, gate)
    ys_m = torch.empty(info["ys_elems"], device="cuda")
    sw.decode_all_layers(xs_p, ys_m)
    torch.cuda.synchronize()
    assert PT.allclose_frac_fail(ys_m.cpu().numpy(), ys_all.cpu().numpy()) == 0.0
    with pytest.raises(L.LswError) as ei:                 # merged ctx: W is no longer pristine
        sw.decode_all_layers_unmerged(xs_p, ys_all, idx, gate)
    assert "STATE" in str(ei.value)


@pytest.mark.parametrize("bad", ["out_of_range", "negative", "duplicate", "nan_gate"])
def test_unmerged_decode_invalid_decision_latches_and_drops_lora(bad):
    """An invalid decision (e.g. idx = -1 from non-finite router logits) is
    never used to index A or B: every CTA validates it, the LoRA terms are
    dropped (y = W x, Eq. 3 on the pristine W) and LSW_DEV_* is latched."""
    cfg = synth.get_config("mini")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    xs = synth.gen_xs(cfg, "cuda")
    idx = torch.tensor([1, 2], dtype=torch.int32, device="cuda")
    gate = torch.tensor([0.75, 0.25], dtype=torch.float32, device="cuda")
    if bad == "out_of_range":
        idx[1] = cfg.n_experts
    elif bad == "negative":
        idx[0] = -1
    elif bad == "duplicate":
        idx[1] = 1
    else:
        gate[0] = float("nan")
    for gi, grp in enumerate(synth.GROUPS):
        n_out = sum(cfg.kind_shape(kd)[0] for kd in grp)
        y = torch.full((n_out,), float("nan"), device="cuda")
        sw.decode_group_unmerged(0, gi, xs[(0, gi)], y, idx, gate)
        torch.cuda.synchronize()
        ref = np.concatenate([O.gemv(_f64(W[kd][0]), _f64(xs[(0, gi)])) for kd in grp])
        np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=1e-4, atol=1e-4 * float(np.abs(ref).max()))
    assert sw.device_status() == (3 if bad == "nan_gate" else 2)
    assert sw.device_status() == 0
