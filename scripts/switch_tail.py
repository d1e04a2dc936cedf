"""Tail of the plain switch pass: per CTA end time (tuning build, seg_trace slot 510)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth
from paper_2405_17741_b200 import binding
from paper_2405_17741_b200 import harness as H
name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
cfg = synth.get_config(name)
W, A, B, router = H.build_weights(cfg, "cuda")
st = torch.zeros(148, 512, 2, dtype=torch.int32, device="cuda")
with binding.options(seg_trace_buf=st.data_ptr()):
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
X1 = synth.gen_x1(cfg, 12, "cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
rows = []
for t in range(10):
    sw.router_topk(X1[t], idx, gate)
    st.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sw.merge_all_layers(idx, gate); b.record()
    torch.cuda.synchronize()
    if t < 3:
        continue
    S = st.cpu().numpy().view("uint32").astype("int64")
    end = S[:, 510, 0]; smid = S[:, 510, 1] - 1
    end = ((end - end.min()) % (1 << 32))
    rows.append((a.elapsed_time(b), np.median(end), end.max(), smid[np.argsort(end)[-4:]].tolist(), end))
for r in rows:
    print(f"pass {r[0]:.3f} ms  end: last - median {int(r[2] - r[1])} ns, last - first {int(r[2])} ns, latest SMs {r[3]}")
E = np.array([r[4] for r in rows])
print("token-to-token corr of per-CTA end:", [round(float(np.corrcoef(E[i], E[i+1])[0, 1]), 3) for i in range(len(E) - 1)])
