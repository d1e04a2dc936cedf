"""GPU router (K2, Eq. 2; G = Softmax(TopK(.)) P:138) vs the oracle's
exact router (ascending-order fp64 loop, O1) on the edge cases SPEC and the
readings fix (-m gpu):
  * ties go to the lower index (R5): equal logits give S = {0..k-1} and
    g = 1/k each; a tie at the top between two experts orders them by index;
  * k = N selects every expert and g is the full softmax;
  * k = 1 gives g = 1.0 exactly (R4);
  * N = 64 (LSW_MAX_EXPERTS) and the full router widths 4096 / 5120 of the
    BASELINE shapes (the reduction length of the fp64 accumulation, R6).
Indices bit-exact, gates within 1e-6 (SURVEY c.5 step 2)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2405_17741_b200 import harness as H


def _f64(t):
    return t.detach().to("cpu").to(torch.float64).numpy()


def _route(cfg, router_rows=None, x=None, n_tok=16):
    W, A, B, router = H.build_weights(cfg, "cuda")
    if router_rows is not None:
        router_rows(router)                     # edit W_g in place before the ctx borrows it
    sw = H.make_switch(cfg, W, A, B, router)
    X1 = synth.gen_x1(cfg, n_tok, "cuda") if x is None else x
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    Wg = _f64(router)
    out = []
    for t in range(X1.shape[0]):
        sw.router_topk(X1[t], idx, gate)
        torch.cuda.synchronize()
        io, go, _ = O.router(Wg, _f64(X1[t]), cfg.top_k)
        out.append((idx.cpu().tolist(), gate.cpu().numpy().astype(np.float64), io.tolist(), go))
    assert sw.device_status() == 0
    sw.close()
    return out


def _check(out):
    for gi, gg, io, go in out:
        assert gi == io
        np.testing.assert_allclose(gg, go, rtol=0, atol=1e-6)
        assert abs(gg.sum() - 1.0) < 1e-6


@pytest.mark.parametrize("name", ["mini", "mini-k1", "mini-kN", "mini-N64", "mini-r4k4", "wide-d4096",
                                  "wide-d5120"])
def test_router_matches_exact_oracle(name):
    cfg = synth.get_config(name)
    out = _route(cfg, n_tok=16 if cfg.d_model <= 256 else 8)
    _check(out)
    if cfg.top_k == 1:
        assert all(g.tolist() == [1.0] for _, g, _, _ in out)          # exactly 1 (R4)
    if cfg.top_k == cfg.n_experts:
        assert all(sorted(i) == list(range(cfg.n_experts)) for i, _, _, _ in out)


def test_router_all_logits_equal_gives_first_k_and_uniform_gates():
    cfg = synth.get_config("mini-r4k4")          # N = 16, k = 4

    def same_rows(r):
        r[:] = r[0].clone()
    out = _route(cfg, same_rows, n_tok=4)
    _check(out)
    for gi, gg, _, _ in out:
        assert gi == [0, 1, 2, 3]
        assert gg.tolist() == [0.25] * 4


def test_router_zero_input_ties_every_expert():
    cfg = synth.get_config("mini-N64")           # N = 64, k = 2: z = 0 for all 64
    x = torch.zeros(2, cfg.d_model, dtype=cfg.torch_dtype, device="cuda")
    out = _route(cfg, x=x)
    _check(out)
    assert all(gi == [0, 1] and gg.tolist() == [0.5, 0.5] for gi, gg, _, _ in out)


def test_router_tie_at_the_top_orders_by_index():
    cfg = synth.get_config("mini")               # N = 8, k = 2
    X1 = synth.gen_x1(cfg, 6, "cuda")
    Wg0 = _f64(synth.gen_router(cfg, "cuda"))
    top = [int(O.router(Wg0, _f64(X1[t]), 1)[0][0]) for t in range(6)]

    def dup_top(r):
        # a copy of token 0's winning row in expert 7 (or 0): every token whose
        # winner is that row now has two equal maximal logits
        e = top[0]
        r[7 if e != 7 else 0] = r[e].clone()
    out = _route(cfg, dup_top, x=X1)
    _check(out)
    e = top[0]
    twin = 7 if e != 7 else 0
    assert out[0][0] == sorted([e, twin]) and out[0][1].tolist() == [0.5, 0.5]
