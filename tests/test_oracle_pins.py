"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test pins one oracle function to something OTHER than itself: values the
SPEC prints (tests/golden), closed forms, brute force, library routines
(torch / scipy), or exact identities on dyadic inputs whose bit budget is
computed in the test.  A plausible bug (dropped term, wrong sign, wrong index,
transposed operand) fails at least one of them -- see the negative checks.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def bits_needed(max_abs: float, quantum: float) -> int:
    """Significant bits to hold every multiple of ``quantum`` up to ``max_abs``."""
    return int(math.ceil(math.log2(max_abs / quantum + 1)))


# ----------------------------------------------------------------------------- rne (O4)

def test_rne_golden_ties():
    for c in _gold("rne_ties.json")["cases"]:
        got = float(O.rne(np.array([c["xv"]]), c["fmt"])[0])
        exp = math.inf if c["expected"] == "inf" else c["expected"]
        assert got == exp, c


def test_rne_f32_matches_numpy_cast():
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.standard_normal(200000) * 0.02,
                        rng.standard_normal(1000) * 1e30,
                        rng.standard_normal(1000) * 1e-40])
    assert np.array_equal(O.rne(v, "f32"), v.astype(np.float32).astype(np.float64))


def test_rne_bf16_matches_torch_cast_of_f32_values():
    # torch's float32 -> bfloat16 cast is RNE; feed values exact in fp32 so
    # there is no double rounding on the torch side.
    rng = np.random.default_rng(2)
    v32 = (rng.standard_normal(200000) * 0.02).astype(np.float32)
    v32 = np.concatenate([v32, (rng.standard_normal(1000) * 1e-39).astype(np.float32)])
    ref = torch.from_numpy(v32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.rne(v32.astype(np.float64), "bf16"), ref)


def test_rne_identity_and_idempotent():
    v = np.random.default_rng(3).standard_normal(1000)
    assert np.array_equal(O.rne(v, None), v)
    b = O.rne(v, "bf16")
    assert np.array_equal(O.rne(b, "bf16"), b)


# ----------------------------------------------------------------------------- router (O1)

def _route_logits(z, k):
    """Router on prescribed logits: W_g = diag-like embedding, x = 1-hot sums."""
    n = len(z)
    Wg = np.diag(np.asarray(z, np.float64))
    x = np.ones(n)
    return O.router(Wg, x, k)


def test_router_golden_equal_logits():
    g = _gold("spec_gate.json")
    idx, gg, g32 = O.router(np.zeros((g["n_experts"], 8)), np.ones(8), g["top_k"])
    assert idx.tolist() == g["expected_idx"]
    assert gg.tolist() == g["expected_g"]


def test_router_bruteforce_rank_definition():
    # e in S  <=>  #{e' : z_e' > z_e or (z_e' == z_e and e' < e)} < k   (R5)
    rng = np.random.default_rng(4)
    for trial in range(300):
        n = int(rng.integers(1, 17))
        k = int(rng.integers(1, n + 1))
        # coarse integer logits force many ties
        z = rng.integers(-3, 4, size=n).astype(np.float64)
        idx, g, _ = _route_logits(z, k)
        S = {e for e in range(n)
             if sum(1 for f in range(n) if z[f] > z[e] or (z[f] == z[e] and f < e)) < k}
        assert set(idx.tolist()) == S
        # output order: descending gate (== descending logit), ties by index
        assert list(idx) == sorted(S, key=lambda e: (-z[e], e))
        assert np.all(np.diff(g) <= 0)


def test_router_k1_gives_one_and_argmax():
    rng = np.random.default_rng(5)
    for _ in range(50):
        Wg = rng.standard_normal((8, 32))
        x = rng.standard_normal(32)
        idx, g, g32 = O.router(Wg, x, 1)
        assert g.tolist() == [1.0] and g32.tolist() == [1.0]
        assert idx[0] == int(np.argmax(Wg @ x))


def test_router_k_equals_n_is_full_softmax():
    rng = np.random.default_rng(6)
    for _ in range(50):
        n = int(rng.integers(2, 16))
        Wg = rng.standard_normal((n, 24))
        x = rng.standard_normal(24)
        idx, g, _ = O.router(Wg, x, n)
        full = scipy.special.softmax(Wg @ x)
        np.testing.assert_allclose(g, full[idx], rtol=1e-12, atol=0)
        assert sorted(idx.tolist()) == list(range(n))


def test_router_topk_softmax_renormalised_exhaustive():
    # equals an exhaustive sort-and-normalise oracle (scipy softmax of the k best)
    rng = np.random.default_rng(7)
    for _ in range(100):
        Wg = rng.standard_normal((8, 40))
        x = rng.standard_normal(40)
        z = Wg @ x
        k = int(rng.integers(1, 9))
        idx, g, _ = O.router(Wg, x, k)
        best = np.argsort(-z, kind="stable")[:k]
        assert idx.tolist() == best.tolist()
        np.testing.assert_allclose(g, scipy.special.softmax(z[best]), rtol=1e-12)
        assert abs(g.sum() - 1.0) < 1e-12


def test_router_shift_invariance():
    rng = np.random.default_rng(8)
    z = rng.standard_normal(8)
    i1, g1, _ = _route_logits(z, 3)
    i2, g2, _ = _route_logits(z + 1000.0, 3)
    assert i1.tolist() == i2.tolist()
    np.testing.assert_allclose(g1, g2, rtol=1e-9)


def test_router_rejects_nonfinite_and_bad_k():
    with pytest.raises(FloatingPointError):
        O.router(np.array([[np.inf, 0.0]]), np.ones(2), 1)
    with pytest.raises(ValueError):
        O.router(np.ones((4, 2)), np.ones(2), 5)


@pytest.mark.parametrize("name,n_tok", [("toy", 64), ("llama2-7b", 6), ("llama2-13b", 6)])
def test_router_fast_matches_router_indices(name, n_tok):
    """router_fast (numpy matvec) routes every parity test; pin it against the
    ascending-order Python loop of ``router`` at the toy width and at the full
    router widths of the BASELINE shapes (d_model 4096 and 5120; bf16 inputs)."""
    cfg = synth.get_config(name)
    Wg = synth.to_f64_numpy(synth.gen_router(cfg))
    X = synth.to_f64_numpy(synth.gen_x1(cfg, n_tok))
    assert Wg.shape == (cfg.n_experts, cfg.d_model)
    for t in range(n_tok):
        a = O.router(Wg, X[t], cfg.top_k)
        b = O.router_fast(Wg, X[t], cfg.top_k)
        assert a[0].tolist() == b[0].tolist()
        np.testing.assert_allclose(a[1], b[1], rtol=1e-13)
        z = np.sort(b[3])[::-1]
        assert z[cfg.top_k - 1] - z[cfg.top_k] > 1e-9     # margins far above fp64 summation-order noise


# ----------------------------------------------------------------------------- delta / merge

def test_delta_golden_spec_matmul():
    g = _gold("spec_matmul.json")
    A = np.array(g["A"], np.float64)[None]
    B = np.array(g["B"], np.float64)[None]
    assert O.delta(A, B, [(0, 1.0)]).tolist() == g["expected_delta"]


def test_merge_textbook_lora_vs_torch():
    # N = k = 1, g = 1: W + (alpha/r) B A, the textbook LoRA merge (Hu et al.)
    rng = np.random.default_rng(9)
    d_out, d_in, r, scale = 48, 80, 8, 2.0
    W = rng.standard_normal((d_out, d_in))
    A = rng.standard_normal((1, r, d_in))
    B = rng.standard_normal((1, d_out, r))
    got = O.merge(W, A, B, ([0], [1.0]), scale, None)
    ref = (torch.from_numpy(W) + scale * torch.from_numpy(B[0]) @ torch.from_numpy(A[0])).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-14)
    # transposed operands / dropped scale are caught:
    assert not np.allclose(got, W + (B[0] @ A[0]))


def _dyadic_site(seed, N=4, r=4, d_out=24, d_in=40):
    W = synth.dyadic((d_out, d_in), -8, 8, 16, seed)
    A = synth.dyadic((N, r, d_in), -8, 8, 16, seed + 1)
    B = synth.dyadic((N, d_out, r), -8, 8, 16, seed + 2)
    return W, A, B


def test_eq5_concat_identity_dyadic_bitexact():
    # [B_e1 ... B_ek] @ [g1 A_e1; ...; gk A_ek] == sum_j g_j B_ej A_ej  (Eq. 5/6)
    W, A, B = _dyadic_site(10)
    idx, gam = [2, 0, 3], [0.75, 0.25, -0.5]
    # bit budget: |g B A| terms are multiples of 2^-10 (1/16*1/16*1/4), sums bounded
    # by 3 * r * (1/2 * 1/2 * 0.75) -> far below 53 bits.
    assert bits_needed(3 * 4 * 0.5 * 0.5 * 0.75, 2.0 ** -10) < 53
    Bcat = np.concatenate([B[e] for e in idx], axis=1)
    Acat = np.concatenate([g * A[e] for e, g in zip(idx, gam)], axis=0)
    assert np.array_equal(O.delta(A, B, list(zip(idx, gam))), Bcat @ Acat)


def test_eq3_merged_forward_equals_eq2_dyadic_bitexact():
    # (W + DeltaW) x == W x + sum_j g_j B_j (A_j x)  (Eq. 3 vs Eq. 2; north_star pin)
    W, A, B = _dyadic_site(11)
    x = synth.dyadic((W.shape[1],), -4, 4, 4, 12)
    cur = ([1, 3], [0.75, 0.25])
    scale = 2.0
    Wm = O.merge(W, A, B, cur, scale, None)
    lhs = O.gemv(Wm, x)
    rhs = W @ x
    for e, g in zip(*cur):
        rhs = rhs + (scale * g) * (B[e] @ (A[e] @ x))
    assert np.array_equal(lhs, rhs)
    assert np.array_equal(O.unmerged_forward(W, A, B, O.coef_list(cur, None, scale), x), rhs)


def test_eq7_unmerge_inverts_merge_dyadic():
    W, A, B = _dyadic_site(13)
    cur = ([0, 2], [0.75, 0.25])
    Wm = O.merge(W, A, B, cur, 1.0, None)
    assert not np.array_equal(Wm, W)
    assert np.array_equal(O.unmerge(Wm, A, B, cur, 1.0, None), W)


def test_eq7_unmerge_inverts_merge_bf16_store_exact_fit():
    # every stored value fits 8 significant bits: W multiples of 1/8 in [-1,1],
    # A, B in {-1,0,1}/4, r <= 4, one expert with gamma = 1 (SURVEY c.4 recipe)
    rng = np.random.default_rng(14)
    W = rng.integers(-8, 9, size=(16, 32)) / 8.0
    A = rng.integers(-1, 2, size=(1, 4, 32)) / 4.0
    B = rng.integers(-1, 2, size=(1, 16, 4)) / 4.0
    # |delta| <= 4/16, multiples of 1/16; W + delta multiples of 1/16 within [-1.25,1.25]
    assert bits_needed(1.25, 1 / 16) <= 8
    Wm = O.merge(W, A, B, ([0], [1.0]), 1.0, "bf16")
    assert np.array_equal(Wm, W + B[0] @ A[0])
    assert np.array_equal(O.unmerge(Wm, A, B, ([0], [1.0]), 1.0, "bf16"), W)


def test_merge_unmerge_not_bitexact_in_general():
    # (a+b)-b != a for generic floats -- pin that the oracle does
    # not fake exact restoration.
    rng = np.random.default_rng(15)
    W = rng.standard_normal((64, 64)) * 0.02
    A = rng.standard_normal((2, 4, 64)) * 0.1
    B = rng.standard_normal((2, 64, 4)) * 0.1
    cur = ([0, 1], [0.6, 0.4])
    back = O.unmerge(O.merge(W, A, B, cur, 1.0, None), A, B, cur, 1.0, None)
    assert not np.array_equal(back, W)
    np.testing.assert_allclose(back, W, rtol=0, atol=1e-15)


def test_eq10_switch_equals_unmerge_then_merge_dyadic():
    W, A, B = _dyadic_site(16)
    prev = ([1, 2], [0.75, 0.25])
    cur = ([2, 3], [0.5, 0.5])
    scale = 4.0
    W1 = O.merge(W, A, B, prev, scale, None)
    W_sw = O.switch(W1, A, B, prev, cur, scale, None)
    W_two = O.merge(O.unmerge(W1, A, B, prev, scale, None), A, B, cur, scale, None)
    assert np.array_equal(W_sw, W_two)
    assert np.array_equal(W_sw, O.merge(W, A, B, cur, scale, None))
    # negative control: literal Eq. 9 gives P + dW(cur) + dW(prev)
    W_lit = O.switch_literal_eq9(W1, A, B, prev, cur, scale, None)
    assert not np.array_equal(W_lit, W_sw)
    exp_lit = W + O.delta(A, B, O.coef_list(cur, None, scale)) + 2 * O.delta(A, B, O.coef_list(prev, None, scale))
    assert np.array_equal(W_lit, exp_lit)


def test_switch_prev_none_is_merge_and_prev_eq_cur_is_noop():
    W, A, B = _dyadic_site(17)
    cur = ([0, 3], [0.75, 0.25])
    assert np.array_equal(O.switch(W, A, B, None, cur, 2.0, None), O.merge(W, A, B, cur, 2.0, None))
    Wm = O.merge(W, A, B, cur, 2.0, "bf16")
    assert np.array_equal(O.switch(Wm, A, B, cur, cur, 2.0, "bf16"), Wm)


def test_restore_is_textbook_merge_of_pristine_and_ends_any_switch_chain():
    """restore(P, cur) = P + sum_j (alpha/r) g_j B_j A_j (textbook
    LoRA merge, torch fp64) and equals, exactly on dyadic inputs, the end of any
    Eq. 6 / Eq. 10 chain started from P -- i.e. it carries no history."""
    W, A, B = _dyadic_site(21)
    scale = 2.0
    cur = ([2, 0], [0.75, 0.25])
    Pt, At, Bt = (torch.from_numpy(np.asarray(t, np.float64)) for t in (W, A, B))
    ref = Pt.clone()
    for e, g in zip(*cur):
        ref += scale * g * (Bt[e] @ At[e])
    np.testing.assert_allclose(O.restore(W, A, B, cur, scale, None), ref.numpy(), rtol=1e-13, atol=1e-13)
    chain = O.merge(W, A, B, ([1, 3], [0.5, 0.5]), scale, None)
    chain = O.switch(chain, A, B, ([1, 3], [0.5, 0.5]), ([3, 2], [0.625, 0.375]), scale, None)
    chain = O.switch(chain, A, B, ([3, 2], [0.625, 0.375]), cur, scale, None)
    assert np.array_equal(O.restore(W, A, B, cur, scale, None), chain)
    # negative control: restoring from the merged W instead of P adds the delta twice
    assert not np.array_equal(O.restore(chain, A, B, cur, scale, None), chain)


def test_coef_list_signs_and_order():
    cl = O.coef_list(([3, 1], [0.7, 0.3]), ([0, 3], [0.6, 0.4]), 2.0)
    assert cl == [(3, 1.4), (1, 0.6), (0, -1.2), (3, -0.8)]
    lit = O.coef_list_literal_eq9(([3, 1], [0.7, 0.3]), ([0, 3], [0.6, 0.4]), 2.0)
    assert [g for _, g in lit] == [1.4, 0.6, 1.2, 0.8]


# ----------------------------------------------------------------------------- gemv (O6)

def test_gemv_vs_torch_fp64():
    rng = np.random.default_rng(18)
    W = rng.standard_normal((77, 130))
    x = rng.standard_normal(130)
    ref = (torch.from_numpy(W) @ torch.from_numpy(x)).numpy()
    np.testing.assert_allclose(O.gemv(W, x), ref, rtol=1e-13, atol=1e-13)
    assert not np.allclose(O.gemv(W, x)[:-1], ref[1:])      # index shift caught


# ----------------------------------------------------------------------------- drift (O7/O8)

@pytest.mark.parametrize("store,eps_tol", [("bf16", 0.15), ("f32", 0.15)])
def test_drift_random_walk_closed_form(store, eps_tol):
    """drift_T ~= eps1 * sqrt(T): eps1 = rel. Frobenius error of one store
    (SURVEY 0.6 / App. B).  Fused switch trajectory vs the exact shadow."""
    rng = np.random.default_rng(19)
    d_out = d_in = 96
    N, r, k, scale = 8, 16, 2, 1.0
    cfgW = rng.standard_normal((d_out, d_in)) * 0.02
    A = rng.uniform(-1, 1, size=(N, r, d_in)) / math.sqrt(d_in)
    sigma_a = 1 / math.sqrt(3 * d_in)
    B = rng.standard_normal((N, d_out, r)) * (0.25 * 0.02 * math.sqrt(k) / (scale * math.sqrt(r) * sigma_a))
    P = O.rne(cfgW, store)
    W = P.copy()
    prev = None
    T = 400
    eps = []
    for t in range(T):
        idx = rng.choice(N, size=k, replace=False)
        gg = rng.dirichlet(np.ones(k))
        cur = (idx.tolist(), gg.tolist())
        exact_prev = W.copy()
        unrounded = exact_prev + O.delta(A, B, O.coef_list(cur, prev, scale))
        W = O.switch(W, A, B, prev, cur, scale, store)
        eps.append(np.linalg.norm(W - unrounded) / np.linalg.norm(unrounded))
        prev = cur
    exact = P + O.delta(A, B, O.coef_list(prev, None, scale))
    d = O.drift(W, exact)["rel_fro"]
    closed = float(np.sqrt(np.mean(np.square(eps)))) * math.sqrt(T)
    assert abs(d / closed - 1.0) < eps_tol, (d, closed)
    # exact mode does not drift (fp64 shadow stays <= 1e-9)
    W64 = O.rne(cfgW, store)
    p2 = None
    for t in range(50):
        idx = rng.choice(N, size=k, replace=False)
        cur = (idx.tolist(), rng.dirichlet(np.ones(k)).tolist())
        W64 = O.switch(W64, A, B, p2, cur, scale, None)
        p2 = cur
    assert O.drift(W64, O.rne(cfgW, store) + O.delta(A, B, O.coef_list(p2, None, scale)))["rel_fro"] < 1e-9


def test_drift_fields_golden_hand_computed():
    """O8's three fields on a hand-worked 2x2 case (allclose is strict '>' in
    |d| > atol + rtol |exact|, torch.allclose's complement):
      exact [[1, -2], [0.5, 0]], W_T - exact [[0.031, 0.04], [0, -0.011]]
      (0,0): 0.031 > 0.01 + 0.02*1 = 0.03  fails;  (0,1): 0.04 <= 0.05  passes;
      (1,0): 0 passes;  (1,1): 0.011 > 0.01  fails  ->  frac_fail = 2/4;
      max_abs = 0.04;  rel_fro = sqrt(0.031^2 + 0.04^2 + 0.011^2) / sqrt(1 + 4 + 0.25)."""
    exact = np.array([[1.0, -2.0], [0.5, 0.0]])
    d = np.array([[0.031, 0.04], [0.0, -0.011]])
    got = O.drift(exact + d, exact)
    assert got["frac_fail"] == 0.5
    assert abs(got["max_abs"] - 0.04) < 1e-15
    assert abs(got["rel_fro"] - math.sqrt(0.031 ** 2 + 0.04 ** 2 + 0.011 ** 2) / math.sqrt(5.25)) < 1e-15
    # a sign error in the difference, or |exact| replaced by exact, is caught:
    assert O.drift(exact - d, exact)["frac_fail"] == 0.5
    z = np.array([[0.0, 1.0]])
    assert O.drift(z + 0.011, z)["frac_fail"] == 0.5                # 0.011 > 0.01 but <= 0.03
    m = np.array([[-1.0, 2.0]])
    assert O.drift(m - 0.029, m)["frac_fail"] == 0.0                # |exact|, not exact, in the bound


# ----------------------------------------------------------------------------- row sampling (O9)

def test_row_sampled_oracle_is_exact():
    cfg = synth.CONFIGS["toy"]
    W = synth.to_f64_numpy(synth.gen_W(cfg, "gate", 1))
    A = synth.to_f64_numpy(synth.gen_A(cfg, "gate", 1))
    B = synth.to_f64_numpy(synth.gen_B(cfg, "gate", 1))
    prev = ([1, 2], [0.6, 0.4])
    cur = ([3, 1], [0.55, 0.45])
    full = O.switch(W, A, B, prev, cur, 4.0, "f32")
    rows = [0, 5, 63, 64, 127]
    part = O.switch(W[rows], A, B[:, rows, :], prev, cur, 4.0, "f32")
    assert np.array_equal(part, full[rows])


# ----------------------------------------------------------------------------- whole model (Alg. 1)

def test_oracle_model_alg1_sequence_matches_exact_shadow_toy():
    cfg = synth.CONFIGS["toy"]
    Wg = synth.to_f64_numpy(synth.gen_router(cfg))
    X1 = synth.to_f64_numpy(synth.gen_x1(cfg, 20))
    Ws, As, Bs = {}, {}, {}
    for kd in synth.KINDS:
        for l in range(cfg.n_layers):
            Ws[(kd, l)] = synth.to_f64_numpy(synth.gen_W(cfg, kd, l))
            As[(kd, l)] = synth.to_f64_numpy(synth.gen_A(cfg, kd, l))
            Bs[(kd, l)] = synth.to_f64_numpy(synth.gen_B(cfg, kd, l))
    m = O.OracleModel(Wg, Ws, As, Bs, cfg.top_k, cfg.alpha, cfg.rank, "f32")
    for t in range(20):
        idx, g, _ = m.route(X1[t])
        m.merge_all_layers((idx, g))
    for key in Ws:
        exact = Ws[key] + O.delta(As[key], Bs[key], O.coef_list((idx, g), None, cfg.alpha / cfg.rank))
        assert O.drift(m.W[key], exact)["rel_fro"] < 1e-5
    m.unmerge_all_layers()
    for key in Ws:
        assert O.drift(m.W[key], Ws[key])["rel_fro"] < 1e-5
    with pytest.raises(RuntimeError):
        m.unmerge_all_layers()


def test_oracle_model_restore_ends_any_chain_and_unmerges_to_pristine_dyadic():
    """OracleModel.restore_merge_all_layers: on dyadic inputs in
    exact mode, restoring d from the pristine copies equals the end of any
    Eq. 6 / Eq. 10 chain that ends at d (every site), records d as merged (a
    following Eq. 7 unmerge gives P back bit for bit), and a following switch
    is Eq. 10 from d."""
    Ws, As, Bs = {}, {}, {}
    for i, kd in enumerate(("q", "down")):
        W, A, B = _dyadic_site(40 + 3 * i)
        Ws[(kd, 0)], As[(kd, 0)], Bs[(kd, 0)] = W, A, B
    Wg = np.eye(4, 8)
    chain = O.OracleModel(Wg, Ws, As, Bs, 2, 8.0, 4, None)      # scale 2
    rest = O.OracleModel(Wg, Ws, As, Bs, 2, 8.0, 4, None)
    d1, d2, d3 = ([1, 3], [0.5, 0.5]), ([3, 2], [0.625, 0.375]), ([0, 2], [0.75, 0.25])
    for d in (d1, d2):
        chain.merge_all_layers(d)
    rest.merge_all_layers(d3)                                    # some other history
    rest.restore_merge_all_layers(Ws, d2)
    for key in Ws:
        assert np.array_equal(rest.W[key], chain.W[key])
        assert not np.array_equal(rest.W[key], Ws[key])
    assert rest.prev == chain.prev
    rest.merge_all_layers(d3)                                    # Eq. 10 from d2
    chain.merge_all_layers(d3)
    for key in Ws:
        assert np.array_equal(rest.W[key], chain.W[key])
    rest.unmerge_all_layers()
    for key in Ws:
        assert np.array_equal(rest.W[key], Ws[key])
