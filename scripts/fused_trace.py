"""Per-tile pipeline trace of the switch kernel (tuning build only:
python paper_2405_17741_b200/build.py --tuning): %globaltimer stamps of
every role for the first 8192 tiles (a whole pass) of CTAs 0-1, for one plain sweep-order
switch and one fused switch + decode token (7B).  Prints medians of the
per-tile intervals (ns): where a tile's time goes."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_17741_b200 import binding  # noqa: E402
from paper_2405_17741_b200 import harness as H  # noqa: E402

SLOTS = ["w_issue", "a_issue", "mma_operands", "mma_commit", "epi_acc", "epi_w", "epi_done", "store_read"]


def analyse(tr):
    out = {}
    for cta in range(tr.shape[0]):
        t = tr[cta].view("uint32").astype("int64")
        n = int((t[:, 6] != 0).sum())
        if n < 10:
            continue
        t = t[:n]
        t = (t - t[0, 6]) % (1 << 32)          # 32-bit timer: differences modulo the wrap
        t = (t + (1 << 31)) % (1 << 32) - (1 << 31)
        rows = {}
        def med(x):
            return float(statistics.median(x)) if len(x) else None
        rows["period_epi_done"] = med([t[i, 6] - t[i - 1, 6] for i in range(1, n)])
        rows["w_load_latency(issue->epi_w)"] = med([t[i, 5] - t[i, 0] for i in range(n)])
        rows["a_load(issue->mma_operands)"] = med([t[i, 2] - t[i, 1] for i in range(n)])
        rows["mma(operands->commit)"] = med([t[i, 3] - t[i, 2] for i in range(n)])
        rows["commit->epi_acc"] = med([t[i, 4] - t[i, 3] for i in range(n)])
        rows["epi_acc_after_w"] = med([t[i, 4] - t[i, 5] for i in range(n)])
        rows["epi_work(max(acc,w)->done)"] = med([t[i, 6] - max(t[i, 4], t[i, 5]) for i in range(n)])
        rows["store(done->read)"] = med([t[i, 7] - t[i, 6] for i in range(n)])
        rows["w_stage_cycle(issue->store_read)"] = med([t[i, 7] - t[i, 0] for i in range(n)])
        rows["period_w_issue"] = med([t[i, 0] - t[i - 1, 0] for i in range(1, n)])
        rows["frac_tiles_acc_last"] = float(sum(1 for i in range(n) if t[i, 4] > t[i, 5]) / n)
        rows["tiles"] = n
        per = [t[i, 6] - t[i - 1, 6] for i in range(1, n)]
        medp = statistics.median(per)
        big = [x for x in per if x > 2.5 * medp]
        rows["stalls_over_2.5x_median"] = len(big)
        rows["stall_excess_us"] = float(sum(x - medp for x in big) / 1e3)
        rows["all_excess_us"] = float(sum(x - medp for x in per if x > medp) / 1e3)
        rows["pass_us"] = float((t[n - 1, 6] - t[0, 6]) / 1e3)
        # period per eighth of the pass (the kinds come in order in the sweep)
        rows["period_by_eighth"] = [float(statistics.median([t[i, 6] - t[i - 1, 6] for i in range(max(1, n * j // 8), n * (j + 1) // 8)]))
                                    for j in range(8)]
        out[f"cta{cta}"] = rows
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    cfg = synth.get_config(name)
    if len(sys.argv) > 2:
        cfg = cfg.with_(n_layers=int(sys.argv[2]))
    extra = dict(kv.split("=") for kv in sys.argv[3:])        # variant options, e.g. tc_pair=1
    W, A, B, router = H.build_weights(cfg, "cuda")
    tr = torch.zeros(2, 8192, 8, dtype=torch.int32, device="cuda")
    st = torch.zeros(148, 512, 2, dtype=torch.int32, device="cuda")
    with binding.options(trace_buf=tr.data_ptr(), seg_trace_buf=st.data_ptr(), **extra):
        sw = H.make_switch(cfg, W, A, B, router, impl="tc")
    X1 = synth.gen_x1(cfg, 8, "cuda")
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
    ys = torch.empty(sw.info()["ys_elems"], device="cuda")
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
    res = {}
    for t in range(3):
        sw.router_topk(X1[t], idx, gate)
        tr.zero_()
        sw.merge_all_layers(idx, gate)
        torch.cuda.synchronize()
    res["sweep_switch"] = analyse(tr.cpu().numpy())
    if os.environ.get("TRACE_SAVE"):                     # raw stamps for offline analysis
        import numpy as np
        np.save(os.environ["TRACE_SAVE"], tr.cpu().numpy())
    if sw.info()["switch_kernel"] == 3:
        for t in range(3, 6):
            tr.zero_()
            st.zero_()
            sw.decode_token_fused(X1[t], xs, ys, idx, gate)
            torch.cuda.synchronize()
        res["fused"] = analyse(tr.cpu().numpy())
        # segment barrier: per segment, the spread of the CTAs' publish times
        # (their own last tile of the segment done) and the wait each CTA sees
        S = st.cpu().numpy().view("uint32").astype("int64")
        n_cta = int((S[:, 0, 0] != 0).sum())
        S = S[:n_cta]
        nseg = int((S[0, :, 0] != 0).sum())
        ref = S[0, 0, 0]
        S = ((S - ref) % (1 << 32) + (1 << 31)) % (1 << 32) - (1 << 31)
        spread, waits, lag = [], [], []
        for g in range(nseg - 1):
            pub = sorted(S[:, g, 0])
            spread.append(float(pub[-1] - pub[len(pub) // 2]))
            waits.append(float(statistics.median(S[:, g, 1] - S[:, g, 0])))
            lag.append(float(statistics.median(S[:, g, 1]) - pub[-1]))
        res["segments"] = {"ctas": n_cta, "segments": nseg,
                           "publish_spread_last_minus_median_ns": statistics.median(spread),
                           "publish_spread_mean_ns": sum(spread) / len(spread),
                           "median_wait_ns": statistics.median(waits),
                           "wait_after_last_publish_ns": statistics.median(lag),
                           "per_segment_spread_first_8": [round(x) for x in spread[:8]]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
