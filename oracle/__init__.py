"""CPU oracle for the LoRA-Switch hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2405_17741_b200``) never imports it and shares no code with it; the
only shared module is ``synth`` (seeded inputs, no method arithmetic).

Plain, slow, obviously-correct numpy in float64.  Every function cites the
passage of arXiv 2405.17741 (``/root/reference/PAPER.md`` line ``P:n``) it
follows; readings of garbled/silent passages are the R-numbers of DESIGN.md §3.

Two layers:
 (i)  exact fp64 definitions (``store=None``) used by the pins in tests/;
 (ii) a store-precision model (``store="bf16"|"f32"``): every merge / unmerge /
      switch pass rounds W ONCE (RNE) to the storage dtype, which is what an
      ideal in-place device kernel holds after each pass.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): rne -> numpy/torch casts and
hand-computed ties; router -> brute-force rank definition, k=1, k=N (scipy
softmax), equal logits, shift invariance; delta/merge -> textbook LoRA merge
(torch fp64), Eq.5 concatenation identity (dyadic, bit-exact); Eq.3==Eq.2
merged forward (dyadic, bit-exact); Eq.7 unmerge inverts Eq.6 (dyadic); Eq.10
== Eq.7 then Eq.6 (dyadic) with the literal Eq.9 as a failing negative
control; restore-from-pristine -> textbook LoRA merge of P (torch fp64) and ==
the switch chain from P (dyadic); drift closed form eps1*sqrt(T); gemv ->
torch fp64 matmul; TP shard invariance.  No function here is "parity unpinned".
"""
from .lsw_oracle import (  # noqa: F401
    rne, router, router_fast, coef_list, coef_list_literal_eq9, delta, merge, unmerge, switch,
    switch_literal_eq9, restore, gemv, unmerged_forward, drift, OracleModel,
)
