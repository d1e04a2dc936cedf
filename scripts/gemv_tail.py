"""GEMV per-CTA end times per group (tuning build: python paper_2405_17741_b200/build.py --tuning; option gemv_trace_buf): spread of the CTAs' end and its token-to-token correlation."""
import sys, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth
from paper_2405_17741_b200 import binding
from paper_2405_17741_b200 import harness as H
cfg = synth.get_config("llama2-7b")
W, A, B, router = H.build_weights(cfg, "cuda")
tr = torch.zeros(512, dtype=torch.int32, device="cuda")
with binding.options(gemv_trace_buf=str(tr.data_ptr())):
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
for gi, grp in enumerate(synth.GROUPS):
    d_in = cfg.kind_shape(grp[0])[1]
    rows = sum(cfg.kind_shape(k)[0] for k in grp)
    x = torch.randn(d_in, device="cuda").to(torch.bfloat16); y = torch.empty(rows, device="cuda")
    spreads = []; ends = []
    for rep in range(12):
        for l in range(3):                         # back to back, PDL-chained as in a token
            sw.decode_group(l, gi, x, y)
        torch.cuda.synchronize()
        t = tr.cpu().numpy().view(np.uint32).astype(np.int64)
        e = t[:148]; e = (e - e.min()) % (1 << 32)
        spreads.append((int(np.median(e)), int(e.max())))
        ends.append(e)
    E = np.array(ends[2:])
    cor = np.mean([np.corrcoef(E[i], E[i+1])[0, 1] for i in range(len(E) - 1)])
    print("+".join(grp), "end spread (median, max) ns:", spreads[-3:], "token corr", round(float(cor), 3))
