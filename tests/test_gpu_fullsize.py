"""Full-size parity at BASELINE.json's Llama-2-7B shape, in the launch
configuration bench.py times (auto -> tcgen05 switch, persistent grid = #SMs),
on sampled rows the oracle computes one by one (-m gpu).

Row sampling is exact, not statistical (O9): row i of the switched W depends
only on row i of W and B and on all of A.  Rows: 0, 1, 127, 128, 129, the
ragged/last rows, plus seeded random rows, of every adapted kind in layers
{0, 1, 15, 31}.  Tokens 1, 2 and 10 are compared (trajectory, one-step,
divergence); the token's decode GEMV outputs are compared on the same rows.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests import parity as PT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LAYERS = (0, 1, 15, 31)
CHECK_T = (1, 2, 10)


def _rows(d_out, seed):
    base = {0, 1, 127, 128, 129, d_out - 129, d_out - 128, d_out - 1}
    g = np.random.default_rng(seed)
    base |= set(g.choice(d_out, size=16, replace=False).tolist())
    return sorted(r for r in base if 0 <= r < d_out)


@pytest.fixture(scope="module")
def big():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2405_17741_b200 import harness as H
    cfg = synth.get_config("llama2-7b")
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="auto")
    yield cfg, W, A, B, router, sw, H
    sw.close()


def test_llama7b_sampled_rows_trajectory_and_gemv(big):
    cfg, W, A, B, router, sw, H = big
    assert sw.info()["switch_impl"] == "tc"
    store, scale = "bf16", cfg.alpha / cfg.rank
    rows = {kd: _rows(cfg.kind_shape(kd)[0], 7 + i) for i, kd in enumerate(synth.KINDS)}
    f64 = lambda t: t.detach().to("cpu").to(torch.float64).numpy()
    keys = [(kd, l) for kd in synth.KINDS for l in LAYERS]
    P = {(kd, l): f64(W[kd][l][rows[kd]]) for kd, l in keys}
    An = {(kd, l): f64(A[kd][l]) for kd, l in keys}
    Bn = {(kd, l): f64(B[kd][l][:, rows[kd], :]) for kd, l in keys}
    orc = O.OracleModel(f64(router), P, An, Bn, cfg.top_k, cfg.alpha, cfg.rank, store)
    X1 = synth.gen_x1(cfg, 12, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    info = sw.info()
    ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    layout, _ = H.ys_layout(cfg)
    yoff = {(l, kd): off for (l, kd, off, n) in layout}
    xs_host = f64(xs)
    x_per_layer = info["xs_elems"] // cfg.n_layers
    gi_of = {kd: gi for gi, grp in enumerate(synth.GROUPS) for kd in grp}
    x_off = {}
    o = 0
    for gi, grp in enumerate(synth.GROUPS):
        x_off[gi] = o
        o += cfg.kind_shape(grp[0])[1]
    prev = None
    W_prev = None
    for t in range(1, 11):
        if t in CHECK_T:
            W_prev = {(kd, l): f64(W[kd][l][rows[kd]]) for kd, l in keys}
        sw.decode_token(X1[t], xs, ys, idx, gate)       # the bench's launch sequence
        torch.cuda.synchronize()
        io, go, _ = orc.route(f64(X1[t]))
        assert idx.cpu().tolist() == io.tolist()
        np.testing.assert_allclose(gate.cpu().numpy(), go, atol=1e-6, rtol=0)
        cur = (io.tolist(), go.tolist())
        orc.merge_all_layers(cur)
        if t in CHECK_T:
            yh = ys.cpu().numpy()
            for kd, l in keys:
                Wg = f64(W[kd][l][rows[kd]])
                Wo = orc.W[(kd, l)]
                assert PT.allclose_frac_fail(Wg, Wo) == 0.0, (t, kd, l)
                assert PT.divergence(Wg, Wo) <= PT.DIVERGENCE_TOL
                r = PT.one_step_ratio(Wg, W_prev[(kd, l)], An[(kd, l)], Bn[(kd, l)], prev, cur, scale, store)
                assert r <= PT.ONE_STEP_TOL, (t, kd, l, r)
                gi = gi_of[kd]
                x = xs_host[l * x_per_layer + x_off[gi]: l * x_per_layer + x_off[gi] + cfg.kind_shape(kd)[1]]
                y_gpu = yh[yoff[(l, kd)] + np.array(rows[kd])]
                assert PT.allclose_frac_fail(y_gpu, O.gemv(Wo, x)) == 0.0, (t, kd, l)
                np.testing.assert_allclose(y_gpu, O.gemv(Wg, x), rtol=1e-4, atol=1e-4)
        prev = cur
    # end of sequence: unmerge restores the pristine weights within tolerance
    sw.unmerge_all_layers()
    orc.unmerge_all_layers()
    torch.cuda.synchronize()
    for kd, l in keys:
        Wg = f64(W[kd][l][rows[kd]])
        assert PT.allclose_frac_fail(Wg, orc.W[(kd, l)]) == 0.0
        assert PT.allclose_frac_fail(Wg, P[(kd, l)]) == 0.0
    assert sw.device_status() == 0
    # one switch launch per merge/unmerge call: router + switch + 4 GEMVs/layer per token
    assert sw.info()["kernel_launches"] == 10 * (2 + 4 * cfg.n_layers) + 1
