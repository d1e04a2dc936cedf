"""LoRA-Switch oracle (numpy, float64) -- TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py for the import rule and the list of pins.  Notation
follows the paper: x^1 router input, G^1 = Softmax(TopK(W_g x^1)) (Eq. 2,
P:228; G defined at P:138), LoRA_DOWN = A (r x d_in), LoRA_UP = B (d_out x r)
(P:139-140), f = backbone weight W (d_out x d_in), Delta W = B A (R2).
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# Significant bits (incl. the implicit one) of each storage format (R15).
_PREC = {"bf16": 8, "f32": 24}
# Smallest exponent of a normal number; subnormal quantum = 2^(EMIN - PREC + 1).
_EMIN = -126
_EMAX = 127


# ---------------------------------------------------------------------------
# O4: store model -- round-to-nearest-even of an fp64 value to the storage type
# ---------------------------------------------------------------------------

def rne(v, fmt: Optional[str]):
    """RNE of float64 values to ``fmt`` ("bf16": 8 significant bits, "f32": 24),
    returned as float64 holding exactly-representable values.  ``fmt=None`` is
    the identity (exact mode).  Written from the definition: the quantum of the
    binade of |v| is 2^(e - p) where |v| in [2^(e-1), 2^e); values are scaled by
    the quantum (exact: power of two), rounded half-to-even (np.rint), and
    scaled back.  Overflow past the largest finite value gives +-inf."""
    if fmt is None:
        return np.asarray(v, dtype=np.float64)
    p = _PREC[fmt]
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros_like(v)
    nz = (v != 0) & np.isfinite(v)
    _, e = np.frexp(v[nz])                      # |v| = m 2^e, m in [0.5, 1)
    qexp = np.maximum(e - p, _EMIN - p + 1)     # subnormals share the min quantum
    q = np.ldexp(1.0, qexp)
    r = np.rint(v[nz] / q) * q
    maxf = (2.0 - 2.0 ** (1 - p)) * 2.0 ** _EMAX
    r = np.where(np.abs(r) > maxf, np.copysign(np.inf, r), r)
    out[nz] = r
    out[~np.isfinite(v)] = v[~np.isfinite(v)]
    return out


# ---------------------------------------------------------------------------
# O1: pre-gated router, Eq. 2 with G = Softmax(TopK(W_g x))
# ---------------------------------------------------------------------------

def router(Wg: np.ndarray, x1: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Returns (idx int32[k], g float64[k], g rounded to float32 [k]).

    z_e = sum_{c ascending} W_g[e, c] x1[c] in fp64 (R6: products of bf16/fp32
    inputs are exact in fp64).  TopK: order experts by (z desc, e asc) (R5),
    keep the first k.  Softmax over the k selected logits only (R4):
    g_i = exp(z_i - max z_S) / sum_{j in S} exp(z_j - max z_S).
    The output is in selection order, i.e. sorted by descending g (R5)."""
    Wg = np.asarray(Wg, dtype=np.float64)
    x1 = np.asarray(x1, dtype=np.float64)
    n_exp, d = Wg.shape
    if not (1 <= k <= n_exp):
        raise ValueError(f"top_k={k} out of range [1, {n_exp}]")
    z = np.zeros(n_exp, dtype=np.float64)
    for e in range(n_exp):
        acc = 0.0
        row = Wg[e]
        # ascending c; float() keeps the sum in Python fp64 scalars
        for c in range(d):
            acc += float(row[c]) * float(x1[c])
        z[e] = acc
    if not np.all(np.isfinite(z)):
        raise FloatingPointError("non-finite router logits")
    order = sorted(range(n_exp), key=lambda e: (-z[e], e))
    S = order[:k]
    zs = np.array([z[e] for e in S], dtype=np.float64)
    m = zs.max()
    ex = np.array([math.exp(v - m) for v in zs], dtype=np.float64)
    g = ex / ex.sum()
    return np.array(S, dtype=np.int32), g, g.astype(np.float32)


def router_fast(Wg: np.ndarray, x1: np.ndarray, k: int):
    """Same definition as ``router`` with the dot products done by numpy
    (library primitive).  Used when many tokens are routed; tests pin that it
    returns the same indices as ``router``."""
    z = np.asarray(Wg, np.float64) @ np.asarray(x1, np.float64)
    if not np.all(np.isfinite(z)):
        raise FloatingPointError("non-finite router logits")
    order = sorted(range(len(z)), key=lambda e: (-z[e], e))
    S = order[:k]
    zs = z[S]
    ex = np.exp(zs - zs.max())
    g = ex / ex.sum()
    return np.array(S, dtype=np.int32), g, g.astype(np.float32), z


# ---------------------------------------------------------------------------
# O2: coefficient list, Eq. 5 and Eq. 9 corrected (R1)
# ---------------------------------------------------------------------------

Decision = Tuple[Sequence[int], Sequence[float]]   # (idx, g)


def coef_list(cur: Optional[Decision], prev: Optional[Decision], scale: float) -> List[Tuple[int, float]]:
    """[(idx_cur[j], +scale*g_cur[j])] followed by [(idx_prev[j], -scale*g_prev[j])].

    Eq. 5 folds the gate into LoRA_DOWN ("G(x)_i . LoRA_DOWN_i"); the
    LoRA scale alpha/r (R3) is folded with it.  Eq. 9 as printed
    negates BOTH previous factors, whose product re-adds the previous delta;
    the sign belongs on exactly one factor, here on the coefficient (R1)."""
    out: List[Tuple[int, float]] = []
    if cur is not None:
        out += [(int(e), +scale * float(g)) for e, g in zip(*cur)]
    if prev is not None:
        out += [(int(e), -scale * float(g)) for e, g in zip(*prev)]
    return out


def coef_list_literal_eq9(cur: Optional[Decision], prev: Optional[Decision], scale: float):
    """NEGATIVE CONTROL (O10): Eq. 9 read literally, concat(-DOWN^{t-1}, DOWN^t)
    with concat(-UP^{t-1}, UP^t); (-D)(-U) = +DU, so the previous term enters
    with a PLUS sign.  Must fail the switch identity."""
    out: List[Tuple[int, float]] = []
    if cur is not None:
        out += [(int(e), +scale * float(g)) for e, g in zip(*cur)]
    if prev is not None:
        out += [(int(e), (-scale * float(g)) * -1.0) for e, g in zip(*prev)]
    return out


# ---------------------------------------------------------------------------
# O3: Delta W for one adapted matrix (Eq. 4/6 P:249-264, product order R2)
# ---------------------------------------------------------------------------

def delta(A_m: np.ndarray, B_m: np.ndarray, coefs: List[Tuple[int, float]]) -> np.ndarray:
    """Delta[i, c] = sum_{(e, gamma) in list order} gamma * (B_e @ A_e)[i, c].

    A_m: LoRA_DOWN bank [N, r, d_in]; B_m: LoRA_UP bank [N, d_out, r] (rows of
    B_m may be a subset: row i of Delta needs only row i of B).  The product
    B_e @ A_e is a library matmul in fp64 (a step, not a reordering)."""
    A_m = np.asarray(A_m, dtype=np.float64)
    B_m = np.asarray(B_m, dtype=np.float64)
    d_out, d_in = B_m.shape[1], A_m.shape[2]
    D = np.zeros((d_out, d_in), dtype=np.float64)
    for e, gamma in coefs:
        D += gamma * (B_m[e] @ A_m[e])
    return D


# ---------------------------------------------------------------------------
# O5: merge (Eq. 6), unmerge (Eq. 7), fused switch (Eq. 10 / SGMM Eq. 11)
# ---------------------------------------------------------------------------

def merge(W, A_m, B_m, cur: Decision, scale: float, store: Optional[str]) -> np.ndarray:
    """Eq. 6: f* = f + DOWN x UP, one rounding to the storage type."""
    return rne(np.asarray(W, np.float64) + delta(A_m, B_m, coef_list(cur, None, scale)), store)


def unmerge(W, A_m, B_m, prev: Decision, scale: float, store: Optional[str]) -> np.ndarray:
    """Eq. 7: f = f*^{t-1} - DOWN^{t-1} x UP^{t-1}."""
    return rne(np.asarray(W, np.float64) + delta(A_m, B_m, coef_list(None, prev, scale)), store)


def switch(W, A_m, B_m, prev: Optional[Decision], cur: Decision, scale: float,
           store: Optional[str]) -> np.ndarray:
    """Eq. 10, applied in place by SGMM (Eq. 11):
    f*^t = f*^{t-1} + Fused_DOWN x Fused_UP, with Eq. 9's concatenation
    corrected (R1).  ONE rounding per pass, as a fused kernel stores once.
    prev=None is the first decode token: a plain merge (R11)."""
    return rne(np.asarray(W, np.float64) + delta(A_m, B_m, coef_list(cur, prev, scale)), store)


def restore(P, A_m, B_m, cur: Decision, scale: float, store: Optional[str]) -> np.ndarray:
    """SURVEY 8f #1 (the alternative P:266 rejects for memory): rebuild the
    merged weight from the pristine copy P every token, f*^t = P + DOWN^t x UP^t
    (Eq. 6 applied to P), one rounding.  No dependence on earlier tokens."""
    return rne(np.asarray(P, np.float64) + delta(A_m, B_m, coef_list(cur, None, scale)), store)


def switch_literal_eq9(W, A_m, B_m, prev, cur, scale, store):
    """NEGATIVE CONTROL: Eq. 10 with the literal (double-negated) Eq. 9."""
    return rne(np.asarray(W, np.float64) + delta(A_m, B_m, coef_list_literal_eq9(cur, prev, scale)), store)


# ---------------------------------------------------------------------------
# O6: merged-forward decode GEMV, Eq. 3; Eq. 2 unmerged form
# ---------------------------------------------------------------------------

def gemv(W, x) -> np.ndarray:
    """y_i = sum_{c ascending} W[i, c] x[c] in fp64 (Eq. 3, batch 1).  The
    row dot products are a library matvec in fp64."""
    return np.asarray(W, np.float64) @ np.asarray(x, np.float64)


def unmerged_forward(P, A_m, B_m, coefs: List[Tuple[int, float]], x) -> np.ndarray:
    """Eq. 2 for one site without merging: P x + sum_j gamma_j B_j (A_j x)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(P, np.float64) @ x
    for e, gamma in coefs:
        y = y + gamma * (np.asarray(B_m[e], np.float64) @ (np.asarray(A_m[e], np.float64) @ x))
    return y


# ---------------------------------------------------------------------------
# O8: drift of a stored trajectory against the exact shadow (O7)
# ---------------------------------------------------------------------------

def drift(W_T: np.ndarray, W_exact: np.ndarray, atol: float = 1e-2, rtol: float = 2e-2) -> Dict[str, float]:
    """rel_fro = ||W_T - W_exact||_F / ||W_exact||_F, max |.|, and the fraction
    of elements outside allclose(atol, rtol)."""
    W_T = np.asarray(W_T, np.float64)
    W_exact = np.asarray(W_exact, np.float64)
    d = W_T - W_exact
    return {
        "rel_fro": float(np.linalg.norm(d) / np.linalg.norm(W_exact)),
        "max_abs": float(np.abs(d).max()),
        "frac_fail": float(np.mean(np.abs(d) > atol + rtol * np.abs(W_exact))),
    }


# ---------------------------------------------------------------------------
# Whole-model oracle: Alg. 1 over every adapted site
# ---------------------------------------------------------------------------

class OracleModel:
    """Holds the stored trajectory of every adapted weight (optionally only a
    row subset per site -- exact, O9: row i of W* depends only on row i of W
    and B and on all of A) and runs Alg. 1 token by token.

    weights[(kind, layer)] : float64 [rows, d_in]   (stored values)
    A[(kind, layer)]       : float64 [N, r, d_in]
    B[(kind, layer)]       : float64 [N, rows, r]
    """

    def __init__(self, Wg, weights, A, B, top_k: int, alpha: float, rank: int, store: Optional[str]):
        self.Wg = np.asarray(Wg, np.float64)
        self.W = {key: np.array(v, dtype=np.float64) for key, v in weights.items()}
        self.A = {key: np.asarray(v, np.float64) for key, v in A.items()}
        self.B = {key: np.asarray(v, np.float64) for key, v in B.items()}
        self.k = top_k
        self.scale = alpha / rank          # R3
        self.store = store
        self.prev: Optional[Decision] = None

    # Alg. 1 line 1 -- Eq. 2
    def route(self, x1):
        idx, g, g32, _ = router_fast(self.Wg, x1, self.k)
        return idx, g, g32

    # Alg. 1 lines 2-4 -- Eq. 5, 9 (R1), 10; first token is a plain merge (R11)
    def merge_all_layers(self, cur: Decision):
        for key in self.W:
            self.W[key] = switch(self.W[key], self.A[key], self.B[key], self.prev, cur, self.scale, self.store)
        self.prev = (tuple(int(e) for e in cur[0]), tuple(float(g) for g in cur[1]))

    # restore from the pristine copies (R11 state: merged(cur))
    def restore_merge_all_layers(self, P, cur: Decision):
        for key in self.W:
            self.W[key] = restore(P[key], self.A[key], self.B[key], cur, self.scale, self.store)
        self.prev = (tuple(int(e) for e in cur[0]), tuple(float(g) for g in cur[1]))

    # End of sequence -- Eq. 7
    def unmerge_all_layers(self):
        if self.prev is None:
            raise RuntimeError("unmerge with nothing merged")
        for key in self.W:
            self.W[key] = unmerge(self.W[key], self.A[key], self.B[key], self.prev, self.scale, self.store)
        self.prev = None

    # Alg. 1 line 5 -- Eq. 3
    def decode_linear(self, kind: str, layer: int, x) -> np.ndarray:
        return gemv(self.W[(kind, layer)], x)
