"""Per-tile timeline of the prefill pair launch (tuning build: python
paper_2405_17741_b200/build.py --tuning; option pf_trace_buf): for the q|k|v
and gate|up groups of the 7B shape at 512 tokens, each CTA's start, and per
tile the time its accumulator was ready and its epilogue done (us from the
earliest CTA start) -- how the rounds of pair tiles actually end."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    cfg = synth.get_config(name).with_(n_layers=2)
    W, A, B, router = H.build_weights(cfg, "cuda")
    tr = torch.zeros(148 * 16 * 4, dtype=torch.int32, device="cuda")
    idx = torch.empty(T, cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(T, cfg.top_k, dtype=torch.float32, device="cuda")
    X1 = synth.gen_x1(cfg, T, "cuda")
    out = {"config": name, "T": T}
    with binding.options(pf_trace_buf=str(tr.data_ptr())):
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
        for t in range(T):
            sw.router_topk(X1[t], idx[t], gate[t])
        for gi in (0, 2):
            grp = synth.GROUPS[gi]
            d_in = cfg.kind_shape(grp[0])[1]
            rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
            X = torch.randn(T, d_in, device="cuda").to(torch.bfloat16)
            Y = torch.empty(T, rows, device="cuda")
            for _ in range(3):
                sw.prefill_group(1, gi, X, idx, gate, Y)
            torch.cuda.synchronize()
            tr.zero_()
            sw.prefill_group(1, gi, X, idx, gate, Y)
            torch.cuda.synchronize()
            a = tr.view(148, 16, 4).cpu().numpy().astype("int64") & 0xFFFFFFFF
            ctas = [c for c in range(148) if a[c, 0, 0] != 0]
            t0 = min(a[c, 0, 0] for c in ctas)
            recs = []
            for c in ctas:
                units = [(int(a[c, u, 0]), round((a[c, u, 2] - t0) / 1e3, 2), round((a[c, u, 3] - t0) / 1e3, 2))
                         for u in range(1, 16) if a[c, u, 3] != 0]
                recs.append({"cta": c, "sm": int(a[c, 0, 1]), "start_us": round((a[c, 0, 0] - t0) / 1e3, 2),
                             "units": units})
            ends = sorted(r["units"][-1][2] for r in recs if r["units"])
            starts = sorted(r["start_us"] for r in recs)
            n_units = [len(r["units"]) for r in recs]
            out["+".join(grp)] = {"ctas": len(recs), "start_us_min_med_max": [starts[0], starts[len(starts) // 2], starts[-1]],
                                  "end_us_min_med_max": [ends[0], ends[len(ends) // 2], ends[-1]],
                                  "units_per_cta": {str(k): n_units.count(k) for k in sorted(set(n_units))},
                                  "first_unit_ready_us_med": sorted(r["units"][0][1] for r in recs)[len(recs) // 2],
                                  "ctas_detail": recs}
        sw.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
