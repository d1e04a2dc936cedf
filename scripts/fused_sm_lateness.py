"""Is the fused decode's segment lateness a property of the SM?  Tuning build:
per CTA the publish time of each segment (seg_trace) and its SM id (slot 511).
Per token: each SM's mean lateness (publish - segment median) over the
segments; then the correlation of the per-SM lateness between tokens."""
import os, sys, statistics
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth
from paper_2405_17741_b200 import binding
from paper_2405_17741_b200 import harness as H

cfg = synth.get_config("llama2-7b")
W, A, B, router = H.build_weights(cfg, "cuda")
st = torch.zeros(148, 512, 2, dtype=torch.int32, device="cuda")
ADAPT = sys.argv[1] if len(sys.argv) > 1 else "1"
with binding.options(seg_trace_buf=st.data_ptr(), fc_adapt=ADAPT):
    sw = H.make_switch(cfg, W, A, B, router, impl="tc")
X1 = synth.gen_x1(cfg, 30, "cuda")
xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
ys = torch.empty(sw.info()["ys_elems"], device="cuda")
idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
per_tok = []
for t in range(24):
    st.zero_()
    sw.decode_token_fused(X1[t], xs, ys, idx, gate)
    torch.cuda.synchronize()
    if t < 18:
        continue
    S = st.cpu().numpy().view("uint32").astype("int64")
    smid = S[:, 511, 0] - 1
    P = S[:, :127, 0]
    ref = P[0, 0]
    P = ((P - ref) % (1 << 32) + (1 << 31)) % (1 << 32) - (1 << 31)
    med = np.median(P, axis=0)
    late = (P - med[None, :]).mean(axis=1)          # per CTA, ns
    per_sm = np.full(160, np.nan)
    per_sm[smid] = late
    per_tok.append(per_sm)
M = np.array(per_tok)
ok = ~np.isnan(M).any(axis=0)
M = M[:, ok]
cors = [np.corrcoef(M[i], M[i + 1])[0, 1] for i in range(len(M) - 1)]
print("adapt", ADAPT); print("per-SM mean lateness ns: token-to-token correlation", [round(c, 3) for c in cors])
print("median over segments of (last - median) publish ns:", float(np.median((P - med[None, :]).max(axis=0))))
print("spread of per-SM mean lateness (std ns):", [round(float(np.std(m)), 1) for m in M])
avg = M.mean(axis=0)
print("SMs most often late (avg ns):", sorted(zip(avg.round(0).tolist(), np.nonzero(ok)[0].tolist()))[-8:])

# per CTA: lateness vs strip boundaries inside its ranges
G = 148
seg_tiles = [(3 * 32 * 32, 32), (32 * 32, 32), (2 * 86 * 32, 32), (32 * 86, 86)] * 32
lat_cta = []
S = st.cpu().numpy().view("uint32").astype("int64")
P = S[:, :127, 0]
ref = P[0, 0]
P = ((P - ref) % (1 << 32) + (1 << 31)) % (1 << 32) - (1 << 31)
med = np.median(P, axis=0)
L = P - med[None, :]
cross = np.zeros((G, 127))
for s_, (T, strip) in enumerate(seg_tiles[:127]):
    for b in range(G):
        lo, hi = T * b // G, T * (b + 1) // G
        cross[b, s_] = (hi - 1) // strip - lo // strip     # strip changes inside the range
        cross[b, s_] += 0 if lo % strip == 0 else 0
tiles = np.array([[T * (b + 1) // G - T * b // G for (T, _) in seg_tiles[:127]] for b in range(G)])
print("corr(lateness, strip changes in range):", round(float(np.corrcoef(L.ravel(), cross.ravel())[0, 1]), 3))
print("corr(lateness, tiles in range):", round(float(np.corrcoef(L.ravel(), tiles.ravel())[0, 1]), 3))
smid = S[:, 511, 0] - 1
late_cta = L.mean(axis=1)
order = np.argsort(late_cta)[::-1][:10]
print("latest CTAs (b, smid, ns):", [(int(b), int(smid[b]), int(late_cta[b])) for b in order])
print("smid of CTA b (first 20):", smid[:20].tolist())
