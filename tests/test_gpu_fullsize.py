"""Full-size parity at BASELINE.json's shapes -- Llama-2-7B (configs[1]),
Mistral-7B (configs[2]: GQA k/v 1024 x 4096, d_ff 14336), Llama-2-13B
(configs[3]: r = 32, the fc fold plan with a single B buffer) and two
configs[4] sweep cells that run the switch's per-term modes -- in the launch
configuration bench.py times (auto -> tcgen05 switch, persistent grid = #SMs,
lsw_decode_token), on sampled rows the oracle computes one by one (-m gpu).

Row sampling is exact, not statistical (O9): row i of the switched W depends
only on row i of W and B and on all of A.  Rows: 0, 1, 127, 128, 129, the
ragged/last rows, plus seeded random rows, of every adapted kind in four
layers.  At the check tokens the stored weights are compared with the
oracle's stored trajectory (allclose), with the oracle's pass applied to the
GPU's own previous state (one-step ratio and 1-ulp flip fraction, the per-pass
bars with teeth of tests/parity.py) and by relative Frobenius divergence; the
token's decode GEMV outputs are compared on the same rows.

The 7B case runs the SURVEY c.5 protocol to token 1000 (checks at 1, 2, 10,
100, 1000) and then the R22 drift report: GPU and oracle drift from the exact
P + DeltaW(d_T) must agree within 10 %.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests import parity as PT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# config -> (layers checked, tokens run, check tokens)
CASES = {
    "llama2-7b": ((0, 1, 15, 31), 1000, (1, 2, 10, 100, 1000)),
    "mistral-7b": ((0, 1, 15, 31), 10, (1, 2, 10)),
    "llama2-13b": ((0, 1, 19, 39), 10, (1, 2, 10)),
    # configs[4] sweep cells on the 7B shape in the switch's other modes:
    # per-term accumulators (r = 32, k = 3) and B staged per unit (r = 64, k = 4)
    "sweep-n16-r32-k3": ((0, 31), 10, (1, 2, 10)),
    "sweep-n8-r64-k4": ((0, 31), 10, (1, 2, 10)),
}
# Trajectory divergence at token 1000 with the hi+lo coefficient split of the
# fc fold (R13): ~1e-3 of the elements take a 1-ulp double-rounding
# flip per pass (9.9e-4), after which the two bf16 random walks
# are independent, so ||W_gpu - W_orc|| / ||W_orc|| grows to ~3e-3 by t = 1000
# (measured 3.0e-3, r01).  The bar is the north_star's 1e-2; 5e-3 flags growth
# beyond what the split explains (a per-term fp32 kernel stays near 4e-4).
DIVERGENCE_T1000 = 5e-3


def _rows(d_out, seed):
    base = {0, 1, 127, 128, 129, d_out - 129, d_out - 128, d_out - 1}
    g = np.random.default_rng(seed)
    base |= set(g.choice(d_out, size=16, replace=False).tolist())
    return sorted(r for r in base if 0 <= r < d_out)


def _f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize_sampled_rows_trajectory_and_gemv(name):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2405_17741_b200 import harness as H
    layers, n_tok, check_t = CASES[name]
    cfg = synth.get_config(name)
    W, A, B, router = H.build_weights(cfg, "cuda")
    sw = H.make_switch(cfg, W, A, B, router, impl="auto")
    try:
        _run(cfg, W, A, B, router, sw, H, layers, n_tok, check_t)
    finally:
        sw.close()
        del W, A, B, router
        torch.cuda.empty_cache()


def _run(cfg, W, A, B, router, sw, H, layers, n_tok, check_t):
    assert sw.info()["switch_impl"] == "tc"
    store, scale = "bf16", cfg.alpha / cfg.rank
    rows = {kd: _rows(cfg.kind_shape(kd)[0], 7 + i) for i, kd in enumerate(synth.KINDS)}
    keys = [(kd, l) for kd in synth.KINDS for l in layers]
    P = {(kd, l): _f64(W[kd][l][rows[kd]]) for kd, l in keys}
    An = {(kd, l): _f64(A[kd][l]) for kd, l in keys}
    Bn = {(kd, l): _f64(B[kd][l][:, rows[kd], :]) for kd, l in keys}
    orc = O.OracleModel(_f64(router), P, An, Bn, cfg.top_k, cfg.alpha, cfg.rank, store)
    X1 = synth.gen_x1(cfg, n_tok + 1, "cuda")
    X1h = _f64(X1)
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    info = sw.info()
    ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    layout, _ = H.ys_layout(cfg)
    yoff = {(l, kd): off for (l, kd, off, n) in layout}
    xs_host = _f64(xs)
    x_per_layer = info["xs_elems"] // cfg.n_layers
    gi_of = {kd: gi for gi, grp in enumerate(synth.GROUPS) for kd in grp}
    x_off, o = {}, 0
    for gi, grp in enumerate(synth.GROUPS):
        x_off[gi] = o
        o += cfg.kind_shape(grp[0])[1]
    gpu_rows = lambda: {(kd, l): _f64(W[kd][l][rows[kd]]) for kd, l in keys}
    prev = None
    W_prev = None
    same_prev, union, prev_set = 0, [], None
    worst = {"div": 0.0, "one_step": 0.0, "step_flip": 0.0}
    for t in range(1, n_tok + 1):
        if t in check_t:
            W_prev = gpu_rows()
        sw.decode_token(X1[t], xs, ys, idx, gate)       # the bench's launch sequence
        io, go, _ = orc.route(X1h[t])
        cur = (io.tolist(), go.tolist())
        orc.merge_all_layers(cur)
        s = set(cur[0])
        if prev_set is not None:
            same_prev += s == prev_set
            union.append(len(s | prev_set))
        prev_set = s
        if t in check_t or t % 50 == 0:
            torch.cuda.synchronize()
            assert idx.cpu().tolist() == io.tolist(), f"token {t}: router indices differ"
            np.testing.assert_allclose(gate.cpu().numpy(), go, atol=1e-6, rtol=0)
        if t in check_t:
            yh = ys.cpu().numpy()
            Wnow = gpu_rows()
            for kd, l in keys:
                Wg, Wo = Wnow[(kd, l)], orc.W[(kd, l)]
                assert PT.allclose_frac_fail(Wg, Wo) == 0.0, (t, kd, l)
                div = PT.divergence(Wg, Wo)
                assert div <= (DIVERGENCE_T1000 if t >= 1000 else PT.DIVERGENCE_TOL), (t, kd, l, div)
                args = (Wg, W_prev[(kd, l)], An[(kd, l)], Bn[(kd, l)], prev, cur, scale, store)
                r = PT.one_step_ratio(*args)
                assert r <= PT.ONE_STEP_TIGHT, (t, kd, l, r)
                fl = PT.one_step_flip_frac(*args)
                assert fl <= PT.STEP_FLIP_TOL, (t, kd, l, fl)
                worst["div"] = max(worst["div"], div)
                worst["one_step"] = max(worst["one_step"], r)
                worst["step_flip"] = max(worst["step_flip"], fl)
                gi = gi_of[kd]
                x = xs_host[l * x_per_layer + x_off[gi]: l * x_per_layer + x_off[gi] + cfg.kind_shape(kd)[1]]
                y_gpu = yh[yoff[(l, kd)] + np.array(rows[kd])]
                assert PT.allclose_frac_fail(y_gpu, O.gemv(Wo, x)) == 0.0, (t, kd, l)
                np.testing.assert_allclose(y_gpu, O.gemv(Wg, x), rtol=1e-4, atol=1e-4)
        prev = cur
    print(f"{cfg.name}: worst {worst}; same-experts-as-prev {same_prev / max(1, n_tok - 1):.4f}, "
          f"mean union {np.mean(union):.3f}")
    if n_tok >= 1000:
        # R22 drift: GPU and oracle trajectories vs the exact P + DeltaW(d_T)
        Wnow = gpu_rows()
        g_all, o_all, e_all = [], [], []
        for key in keys:
            exact = P[key] + O.delta(An[key], Bn[key], O.coef_list(prev, None, scale))
            g_all.append(Wnow[key].ravel())
            o_all.append(orc.W[key].ravel())
            e_all.append(exact.ravel())
        g_all, o_all, e_all = map(np.concatenate, (g_all, o_all, e_all))
        dg, do = O.drift(g_all, e_all), O.drift(o_all, e_all)
        print(f"{cfg.name} drift at T={n_tok}: gpu {dg}, oracle {do}")
        assert 0.9 <= dg["rel_fro"] / do["rel_fro"] <= 1.1, (dg, do)
        assert 5e-3 < do["rel_fro"] < 0.1                 # the bf16 random walk is there (eps1 sqrt(T))
        # the router's routing statistics are those of independent uniform routing
        # (1/C(8,2) = 0.036 same-set tokens, E|S u S'| = 2k - k^2/N = 3.5)
        assert 0.01 < same_prev / (n_tok - 1) < 0.08 and 3.3 < np.mean(union) < 3.7
    # end of sequence: unmerge restores the pristine weights within tolerance
    sw.unmerge_all_layers()
    orc.unmerge_all_layers()
    torch.cuda.synchronize()
    Wnow = gpu_rows()
    for key in keys:
        assert PT.allclose_frac_fail(Wnow[key], orc.W[key]) == 0.0
        assert PT.divergence(Wnow[key], orc.W[key]) <= PT.DIVERGENCE_TOL
        if n_tok < 1000:
            # (after 1000 passes the stored trajectory has drifted ~5 % from P -- the
            # oracle's as much as the GPU's, measured above -- and a few elements
            # of ~0.02 leave the 1e-2 atol band: compared with the oracle only)
            assert PT.allclose_frac_fail(Wnow[key], P[key]) == 0.0
    assert sw.device_status() == 0
    # one switch launch per merge/unmerge call: router + switch + 4 GEMVs/layer per token
    assert sw.info()["kernel_launches"] == n_tok * (2 + 4 * cfg.n_layers) + 1
