"""Per-tile pipeline timeline of the tensor-core switch (LSW_TC_TRACE=1): runs a
few switches at a BASELINE shape, reads the trace (include/lsw_debug.h) of CTAs
0, 49, 98, 147 and prints, per CTA, its span and per-tile rate in windows, plus
median intervals between pipeline events."""
import os
import sys

os.environ["LSW_TC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

EV = ["W_issued", "A_issued", "A_full", "MMA_start", "MMA_done", "EPI_wfull", "EPI_acc0", "stage_free",
      "EPI_done", "MMA_acc0", "MMA_issued0", "EPI_sub0_done", "A_begin", "A_waited", "EPI_acc1", "MMA_issued1"]
if os.environ.get("LSW_TRACE_LIB"):          # A/B against another build of the library
    from paper_2405_17741_b200 import binding as _B
    _B._LIB = _B.load_library(os.environ["LSW_TRACE_LIB"], strict=False)
cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b")
W, A, B, router = H.build_weights(cfg, "cuda")
sw = H.make_switch(cfg, W, A, B, router, impl="tc")
X1 = synth.gen_x1(cfg, 6, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
for t in range(6):
    sw.router_topk(X1[t], idx, gate)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sw.merge_all_layers(idx, gate)
    e1.record()
    torch.cuda.synchronize()
    print(f"token {t} idx {idx.cpu().tolist()} switch {e0.elapsed_time(e1):.3f} ms")
tr = sw.debug_switch_trace().astype(np.int64)
t_begin = tr[tr > 0].min()
for slot, cta in enumerate((0, 49, 98, 147)):
    T = tr[slot]
    ok = (T[:, EV.index("EPI_done")] > 0)
    T = T[ok]
    if len(T) < 10:
        continue
    done = T[:, EV.index("EPI_done")]
    print(f"CTA {cta}: tiles {len(T)}  first W {(T[0, 0] - t_begin) / 1e3:.1f} us  last done "
          f"{(done[-1] - t_begin) / 1e3:.1f} us  mean us/tile {np.mean(np.diff(done)) / 1e3:.3f}")
    n = len(done)
    for w0 in range(0, n, max(1, n // 6)):
        w1 = min(n - 1, w0 + max(1, n // 6))
        if w1 > w0:
            print(f"   tiles {w0:5d}-{w1:5d}: us/tile {(done[w1] - done[w0]) / (w1 - w0) / 1e3:.3f}")
    d = lambda a, b: np.median(T[:, EV.index(b)] - T[:, EV.index(a)]) / 1e3
    for a, b in [("W_issued", "EPI_wfull"), ("A_issued", "A_full"), ("MMA_start", "A_full"), ("A_begin", "A_waited"), ("A_waited", "A_issued"), ("MMA_issued0", "MMA_issued1"), ("MMA_issued1", "MMA_done"),
                 ("MMA_issued1", "EPI_acc1"), ("EPI_sub0_done", "EPI_acc1"), ("EPI_acc1", "EPI_done"), ("A_full", "MMA_acc0"),
                 ("MMA_acc0", "MMA_issued0"), ("MMA_issued0", "MMA_done"),
                 ("MMA_issued0", "EPI_acc0"), ("EPI_acc0", "EPI_sub0_done"), ("EPI_sub0_done", "EPI_done"),
                 ("EPI_done", "stage_free")]:
        print(f"   {a:>13s} -> {b:<13s} median {d(a, b):8.3f} us")
    nxt = np.median(T[1:, EV.index("MMA_start")] - T[:-1, EV.index("MMA_done")]) / 1e3
    print(f"   MMA_done(t) -> MMA_start(t+1) median {nxt:8.3f} us;  MMA_start period "
          f"{np.median(np.diff(T[:, EV.index('MMA_start')])) / 1e3:.3f} us")
    w_wait = T[1:, EV.index("EPI_wfull")] - T[:-1, EV.index("EPI_done")]
    a_wait = T[:, EV.index("EPI_acc0")] - T[:, EV.index("EPI_wfull")]
    print(f"   epilogue idle per tile: waiting W mean {np.mean(w_wait) / 1e3:.3f} us, "
          f"waiting acc mean {np.mean(a_wait) / 1e3:.3f} us")
