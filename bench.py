#!/usr/bin/env python
"""Benchmark of the LoRA-Switch hot path on B200 (driver contract).

One STEP = one decode token of Alg. 1 over every adapted linear of
every layer: pre-gated router (Eq. 2) -> ONE all-layer switch launch (Eq. 10)
-> the batch-1 decode GEMVs on the merged weights (Eq. 3), 4 grouped GEMV
launches per layer (+ NCCL allreduce of the row-parallel partial sums under TP).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama2-7b]
                  [--impl ours|reference] [--switch-impl auto|tc|simt]

value    = algorithmic HBM bytes of the whole token (all ranks) / device time
           per token, GB/s (metric: "merge+unmerge HBM GB/s vs peak; decode
           ms/token at Llama-2-7B shape"); ms_per_step = decode ms/token.
roofline = the dominant kernel (the fused switch): algorithmic bytes per launch
           / its CUDA-event duration on the launching stream, vs the measured
           copy peak in MEASURED_PEAKS.json.
e2e      = the same metric through lsw_decode_token_host (host pinned buffers,
           H2D of the token inputs and D2H of all outputs inside the timed region).
cpu_baseline / --impl reference = the numpy fp64 oracle (oracle/, untuned) on a
           bounded sample of the same workload, on this host's cores.
Inputs (13 GB of weights for 7B) are far larger than the 126 MB L2, so no flush
is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "merge+unmerge HBM GB/s vs peak; decode ms/token at Llama-2-7B shape"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _workload(cfg, n):
    return (f"{cfg.name}: {cfg.n_layers} layers, d_model {cfg.d_model}, d_ff {cfg.d_ff}, "
            f"q/kv heads {cfg.n_heads}/{cfg.n_kv_heads}, 7 adapted linears per layer, "
            f"{cfg.n_experts} experts r={cfg.rank} top-{cfg.top_k}, alpha {cfg.alpha:g}, {cfg.dtype}; "
            f"1 decode token per step (router + 1 switch launch + {4 * cfg.n_layers} GEMV launches)"
            + (f", TP={n}" if n > 1 else ""))


class ClockSampler:
    """nvidia-smi clocks during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        sm, mx, reasons = [], [], set()
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx.append(float(p[2]))
                except ValueError:
                    continue
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for nm, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except Exception:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


SWITCH_KERNELS = {3: "switch_fc_kernel [fold: folded coefficients, one accumulator per tile]",
                  4: "switch_fc_kernel [per-term accumulators, B per strip]",
                  5: "switch_fc_kernel [per-term accumulators, B per unit]",
                  7: "switch_fc_kernel [fold, (hi, lo) B strip in TMEM: one accumulator per tile]"}


def _ncu_traffic(cfg, info):
    """DRAM traffic per switch launch from the committed ncu capture
    (profiles/ncu_switch_traffic.json), scaled from its layer count to this
    config's; None if the capture is missing or for another shape/impl."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_switch_traffic.json")) as f:
            d = json.load(f)
        if d.get("config") != cfg.name or d.get("switch_impl") != info["switch_impl"]:
            return None
        if d.get("switch_kernel") not in (None, info.get("switch_kernel")):
            return None
        return d["dram_bytes_per_layer"] * cfg.n_layers
    except Exception:
        return None


def _drift_profile(cfg):
    """R22 drift of the committed 1000-token report (scripts/drift_report.py,
    GPU and oracle side by side on sampled rows) for this config, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "drift_%s.json" % cfg.name)) as f:
            d = json.load(f)
        return {"tokens": d["tokens"],
                "switch_rel_fro_gpu": d["switch"]["gpu_vs_exact"]["rel_fro"],
                "switch_rel_fro_oracle": d["switch"]["oracle_vs_exact"]["rel_fro"],
                "switch_ratio": d["switch"]["drift_ratio_gpu_over_oracle"],
                "switch_gpu_vs_oracle_rel_fro": d["switch"]["gpu_vs_oracle"]["rel_fro"],
                "cycles_rel_fro_gpu": d["cycles"]["gpu_vs_pristine"]["rel_fro"],
                "cycles_ratio": d["cycles"]["drift_ratio_gpu_over_oracle"],
                "source": "profiles/drift_%s.json (scripts/drift_report.py)" % cfg.name}
    except Exception:
        return None


def _host_cpu():
    """Host identity for the CPU baseline (SURVEY d.6): model, threads allowed,
    the BLAS / OpenMP thread setting."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("user_api"), "lib": i.get("internal_api"), "threads": i.get("num_threads")}
                for i in threadpool_info()]
    except Exception:
        pass
    return {"model": model, "affinity_cpus": len(os.sched_getaffinity(0)),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"), "threadpools": blas}


# ----------------------------------------------------------------------------- CPU oracle leg

_SAMPLE_CACHE = {}


def oracle_sample(cfg, seconds_budget: float = 15.0):
    """Time the untuned numpy oracle on a bounded sample of the workload: the
    switch (Eq. 10, one rounding, bf16 store) and the GEMV (Eq. 3) on R rows of
    every adapted matrix of layer 0, plus one router call.  Returns GB/s of
    algorithmic bytes (same accounting as the GPU) and the sample description.
    The seeded sample inputs are generated once per process (not timed)."""
    import torch

    import oracle as O
    import synth
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = 1
    store = "bf16" if cfg.dtype == "bf16" else "f32"
    scale = cfg.alpha / cfg.rank
    s = cfg.elem_bytes
    rows = 256
    if cfg.name not in _SAMPLE_CACHE:
        Wg = synth.gen_router(cfg).double().numpy()
        x1 = synth.gen_x1(cfg, 2).double().numpy()
        mats = []
        for kd in synth.KINDS:
            d_out, d_in = cfg.kind_shape(kd)
            R = min(rows, d_out)
            W = synth.gen_W(cfg, kd, 0)[:R].double().numpy()
            A = synth.gen_A(cfg, kd, 0).double().numpy()
            B = synth.gen_B(cfg, kd, 0)[:, :R].double().numpy()
            x = torch.randn(d_in).to(cfg.torch_dtype).double().numpy()
            mats.append((kd, W, A, B, x))
        _SAMPLE_CACHE[cfg.name] = (Wg, x1, mats)
    Wg, x1, mats = _SAMPLE_CACHE[cfg.name]
    t0 = time.perf_counter()
    nbytes = 0.0
    passes = 0
    prev = None
    while True:
        idx, g, _ = O.router(Wg, x1[passes % 2], cfg.top_k)
        nbytes += s * cfg.n_experts * cfg.d_model + s * cfg.d_model
        cur = (idx.tolist(), g.tolist())
        for kd, W, A, B, x in mats:
            R, d_in = W.shape
            W[:] = O.switch(W, A, B, prev, cur, scale, store)
            O.gemv(W, x)
            K = 2 * cfg.top_k * cfg.rank
            nbytes += 2 * s * R * d_in + s * K * (R + d_in) + s * R * d_in + s * d_in + 4 * R
        prev = cur
        passes += 1
        if time.perf_counter() - t0 > seconds_budget:
            break
    dt = time.perf_counter() - t0
    sample = (f"{passes} pass(es) of router + switch + GEMV on the first {rows} rows of each of the 7 "
              f"adapted matrices of layer 0 ({cfg.name}), numpy fp64 with bf16 RNE store model")
    return nbytes / dt / 1e9, sample, cores, dt


def run_reference(args, cfg):
    """--impl reference: the oracle as it stands, on this host, same metric."""
    import torch.distributed as dist  # noqa: F401
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    samples = None
    cores = 1
    total = 0.0
    for i in range(args.warmup + args.steps):
        v, sample, cores, dt = oracle_sample(cfg, seconds_budget=args.ref_seconds)
        if i >= args.warmup:
            vals.append(v)
            total += dt
        samples = sample
    val = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / max(1, args.steps),
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic", "config": {"workload": _workload(cfg, 1)},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": samples},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2405_17741_b200 import harness as H
    from paper_2405_17741_b200.binding import LoraSwitch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (launch with torchrun for N>1)")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = "cuda"

    W, A, B, router = H.build_weights(cfg, dev, rank, world)
    sw = H.make_switch(cfg, W, A, B, router, impl=args.switch_impl, tp_rank=rank, tp_size=world)
    if world > 1:
        uid = [LoraSwitch.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sw.attach_nccl(uid[0])
    info = sw.info()
    n_tok = args.warmup + args.steps
    X1 = synth.gen_x1(cfg, n_tok + 8, dev)
    xs = H.pack_xs(cfg, synth.gen_xs(cfg, dev), rank, world)
    ys = torch.empty(info["ys_elems"], dtype=torch.float32, device=dev)
    idx = torch.empty(cfg.top_k, dtype=torch.int32, device=dev)
    gate = torch.empty(cfg.top_k, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    tb = H.token_bytes(cfg, world)

    # decode token loop: events bracket the switch launch on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(n_tok)]
    # The timed step is one lsw_decode_token call (router + switch + GEMVs, all
    # enqueued from C); the per-kernel breakdown below repeats the same launch
    # sequence call by call with events around the switch.
    def token(t):
        sw.decode_token(X1[t], xs, ys, idx, gate, stream)

    torch.cuda.synchronize()
    for t in range(args.warmup):
        token(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = sw.info()["kernel_launches"]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_start.record(stream)
        for t in range(args.warmup, n_tok):
            token(t)
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = sw.info()["kernel_launches"] - launches0
    ms_total = t_start.elapsed_time(t_end)
    # routing statistics of the timed tokens (SURVEY d.2): their decisions again
    # through the router kernel, read back after the timed region
    decs = []
    for t in range(args.warmup - 1, n_tok):
        sw.router_topk(X1[t], idx, gate, stream)
        decs.append(idx.clone())
    decs = torch.stack(decs).cpu().tolist()
    sets = [set(d) for d in decs]
    same = [sets[i] == sets[i - 1] for i in range(1, len(sets))]
    union = [len(sets[i] | sets[i - 1]) for i in range(1, len(sets))]
    routing = {"tokens": len(same), "same_experts_as_prev": sum(same) / max(1, len(same)),
               "mean_union_size": sum(union) / max(1, len(union)),
               "expected_independent_uniform": {"same": 1.0 / math.comb(cfg.n_experts, cfg.top_k),
                                                "union": 2 * cfg.top_k - cfg.top_k ** 2 / cfg.n_experts}}
    if world > 1:
        tt = torch.tensor([ms_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    clocks = clk.summary()

    # kernel breakdown: router | switch | GEMVs, events on the launching stream
    sw_ms, gemv_ms = [], []
    for t in range(args.steps):
        e0, e1, e2 = ev[t]
        sw.router_topk(X1[t + 1], idx, gate, stream)
        e0.record(stream)
        sw.merge_all_layers(idx, gate, stream)
        e1.record(stream)
        sw.decode_all_layers(xs, ys, stream)
        e2.record(stream)
    torch.cuda.synchronize()
    for t in range(args.steps):
        e0, e1, e2 = ev[t]
        sw_ms.append(e0.elapsed_time(e1))
        gemv_ms.append(e1.elapsed_time(e2))
    sw_med = statistics.median(sw_ms)
    gemv_med = statistics.median(gemv_ms)

    # merge-only / unmerge-only passes (Eq. 6 / Eq. 7)
    mg_ms, um_ms = [], []
    for t in range(min(args.steps, 10)):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        sw.unmerge_all_layers(stream)
        b.record(stream)
        sw.merge_all_layers(idx, gate, stream)
        c.record(stream)
        torch.cuda.synchronize()
        um_ms.append(a.elapsed_time(b))
        mg_ms.append(b.elapsed_time(c))

    # restore-from-pristine switch: W <- RNE(P + Delta(d_t)), same
    # 4 B/element as the fused switch; P = a copy of the weights as they are now
    # (timing only: the bytes and the kernel do not depend on P's values)
    rs_ms = []
    if not args.no_restore:
        P = {kd: W[kd].clone() for kd in synth.KINDS}
        sw.attach_pristine(P)
        for t in range(min(args.steps, 10)):
            sw.router_topk(X1[t], idx, gate, stream)
            a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            a.record(stream)
            sw.restore_merge_all_layers(idx, gate, stream)
            b.record(stream)
            torch.cuda.synchronize()
            rs_ms.append(a.elapsed_time(b))
        del P

    # launch-count ablation (the paper's Tab. 6 "simple merge"):
    # the Eq. 6 merge as 1 launch vs one launch per matrix (7 L), eager and
    # replayed from a CUDA graph (each graph = merge + the single unmerge)
    abl = None
    if world == 1 and info["switch_impl"] == "tc":
        sw.unmerge_all_layers(stream)

        def _time(fn, n=5):
            ms = []
            for _ in range(n):
                a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            return statistics.median(ms)

        single = lambda: sw.merge_all_layers(idx, gate, stream)
        per_mat = lambda: sw.debug_merge_per_matrix(idx, gate, stream)
        abl = {"launches_single": 1, "launches_per_matrix": 7 * cfg.n_layers}
        for key, fn in (("single", single), ("per_matrix", per_mat)):
            ms = []
            for _ in range(5):
                a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
                sw.unmerge_all_layers(stream)
            abl[key + "_ms"] = statistics.median(ms)
        gs = torch.cuda.Stream()
        torch.cuda.synchronize()
        # graphs: capture merge + unmerge on the capture stream
        for key, merge in (("single", lambda st: sw.merge_all_layers(idx, gate, st)),
                           ("per_matrix", lambda st: sw.debug_merge_per_matrix(idx, gate, st))):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                merge(gs)
                sw.unmerge_all_layers(gs)
            abl[key + "_graph_merge_plus_unmerge_ms"] = _time(g.replay)
            del g
        um_only = _time(lambda: (sw.merge_all_layers(idx, gate, stream), sw.unmerge_all_layers(stream)))
        abl["single_eager_merge_plus_unmerge_ms"] = um_only

    # fused switch + decode: router + ONE launch that switches and
    # computes the GEMVs in decoder order (4 B/element, 4L segment barriers)
    fu_ms = []
    fused_ok = False
    if world == 1 and info["switch_impl"] == "tc":
        # (the fused launch is the fold mode's fused build -- an untimed
        # warm-up token first builds its segment table)
        try:
            sw.decode_token_fused(X1[0], xs, ys, idx, gate, stream)
            torch.cuda.synchronize()
            fused_ok = True
        except Exception as e:  # noqa: BLE001  (LSW_E_UNSUPPORTED for this shape)
            print(f"[bench] fused decode not timed: {e}", file=sys.stderr)
    if fused_ok:
        for t in range(min(args.steps, 10)):
            a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            a.record(stream)
            sw.decode_token_fused(X1[t + 1], xs, ys, idx, gate, stream)   # X1[0] was the warm-up
            b.record(stream)
            torch.cuda.synchronize()
            fu_ms.append(a.elapsed_time(b))

    # unmerged decode (the honest comparison): router + Eq. 2 on the
    # pristine weights, W read once (2 B/element) instead of switched and read (6)
    un_ms = []   # (TP: the o / down partials are all-reduced by the library)
    if sw.info()["merged"]:
        sw.unmerge_all_layers(stream)
    for t in range(min(args.steps, 10)):
        a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        a.record(stream)
        sw.router_topk(X1[t], idx, gate, stream)
        sw.decode_all_layers_unmerged(xs, ys, idx, gate, stream)
        b.record(stream)
        torch.cuda.synchronize()
        un_ms.append(a.elapsed_time(b))

    # unmerged prefill: a 512-token prompt, every token with its
    # own pre-gated decision, through every group of every layer (Eq. 2; our
    # tcgen05 LoRA-down GEMM, Z build and dense + LoRA-up GEMM per group) --
    # reported, not timed into the decode metric
    pf = None
    if world == 1:
        T_pf = 512
        Xp = synth.gen_x1(cfg, T_pf, dev)
        idx_pf = torch.empty(T_pf, cfg.top_k, dtype=torch.int32, device=dev)
        gate_pf = torch.empty(T_pf, cfg.top_k, dtype=torch.float32, device=dev)
        for t in range(T_pf):
            sw.router_topk(Xp[t], idx_pf[t], gate_pf[t], stream)
        d_ins = sorted({cfg.kind_shape(grp[0])[1] for grp in synth.GROUPS})
        Xg = {d: torch.randn(T_pf, d, device=dev).to(Xp.dtype) for d in d_ins}
        Yp = torch.empty(T_pf * max(sum(cfg.kind_shape(kd)[0] for kd in grp) for grp in synth.GROUPS), device=dev)

        def prefill():
            for l in range(cfg.n_layers):
                for gi, grp in enumerate(synth.GROUPS):
                    rows = sum(cfg.kind_shape(kd)[0] for kd in grp)
                    sw.prefill_group(l, gi, Xg[cfg.kind_shape(grp[0])[1]], idx_pf, gate_pf,
                                     Yp[:T_pf * rows].view(T_pf, rows), stream)
        prefill()
        torch.cuda.synchronize()
        pf_ms = []
        for _ in range(3):
            a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            a.record(stream)
            prefill()
            b.record(stream)
            torch.cuda.synchronize()
            pf_ms.append(a.elapsed_time(b))
        pf_fl = 2.0 * T_pf * cfg.n_layers * sum(
            cfg.kind_shape(kd)[0] * (cfg.kind_shape(kd)[1] + 2 * cfg.n_experts * ((cfg.rank + 15) // 16 * 16))
            + cfg.n_experts * cfg.rank * cfg.kind_shape(kd)[1] for kd in synth.KINDS)
        pf = {"tokens": T_pf, "ms": statistics.median(pf_ms),
              "tokens_per_s": T_pf / (statistics.median(pf_ms) * 1e-3),
              "tflops_issued": pf_fl / (statistics.median(pf_ms) * 1e-3) / 1e12,
              "note": "adapted-linear prefill of all layers on our tcgen05 kernels (dense + LoRA-up in one "
                      "contraction per tile, every expert's LoRA-down); router per token excluded; "
                      "tflops_issued counts the MMA work issued (dense d_in + 2 N rp LoRA-up K + N r LoRA-down)"}

    # end-to-end through the public API with host buffers
    x1h = torch.empty(cfg.d_model, dtype=cfg.torch_dtype).pin_memory()
    xsh = xs.cpu().pin_memory()
    ysh = torch.empty(info["ys_elems"], dtype=torch.float32).pin_memory()
    idxh = torch.empty(cfg.top_k, dtype=torch.int32).pin_memory()
    gh = torch.empty(cfg.top_k, dtype=torch.float32).pin_memory()
    X1h = X1.cpu()
    e2e_steps = max(3, min(args.steps, 20))
    for t in range(2):
        x1h.copy_(X1h[t])
        sw.decode_token_host(x1h, xsh, ysh, idxh, gh, stream)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for t in range(e2e_steps):
        x1h.copy_(X1h[t % X1h.shape[0]])
        sw.decode_token_host(x1h, xsh, ysh, idxh, gh, stream)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    assert sw.device_status(stream) == 0

    # aggregate over ranks: token bytes of all ranks / max time
    tok_bytes_all = tb["token"] * world if world == 1 else None
    if world > 1:
        tt = torch.tensor([tb["token"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tt)
        tok_bytes_all = float(tt.item())
    value = tok_bytes_all / (ms_step * 1e-3) / 1e9
    peak, peak_src = _peaks()
    sw_gbs = tb["switch"] / (sw_med * 1e-3) / 1e9
    res = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, sample, cores, _ = oracle_sample(cfg, seconds_budget=max(args.ref_seconds, 10.0))
            cpu = {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample,
                   "host": _host_cpu()}
        h2d = x1h.numel() * x1h.element_size() + xsh.numel() * xsh.element_size()
        d2h = ysh.numel() * 4 + cfg.top_k * 8
        res = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded random-init weights/adapters of the named shape)",
            "config": {"workload": _workload(cfg, world), "parallelism": f"tp{world}",
                       "l2": "no flush: weights (%.1f GB/GPU) >> 126 MB L2" % (tb["w_elems"] * cfg.elem_bytes / 1e9),
                       "switch_impl": info["switch_impl"], "switch_grid": info["grid"],
                       "switch_tile": [info["tile_m"], info["tile_n"]]},
            "decode_ms_per_token": ms_step,
            "decode_frac_of_roofline": (tb["token"] / (peak * 1e9)) * 1e3 / ms_step,
            "switch_ms": sw_med, "switch_GBps": sw_gbs, "gemv_ms_per_token": gemv_med,
            "gemv_GBps": tb["gemv"] / (gemv_med * 1e-3) / 1e9,
            "merge_GBps": tb["merge"] / (statistics.median(mg_ms) * 1e-3) / 1e9,
            "unmerge_GBps": tb["merge"] / (statistics.median(um_ms) * 1e-3) / 1e9,
            "restore_ms": statistics.median(rs_ms) if rs_ms else None,
            "restore_GBps": tb["merge"] / (statistics.median(rs_ms) * 1e-3) / 1e9 if rs_ms else None,
            "launch_ablation": abl,
            "fused_decode_ms_per_token": statistics.median(fu_ms) if fu_ms else None,
            "unmerged_decode_ms_per_token": statistics.median(un_ms) if un_ms else None,
            "unmerged_decode_GBps": (tb["unmerged_token"] / (statistics.median(un_ms) * 1e-3) / 1e9
                                     if un_ms else None),
            "prefill": pf,
            "decode_frac_of_nominal_8TBps": (tb["token"] / 8.0e12) * 1e3 / ms_step,
            "routing": routing,
            "drift": _drift_profile(cfg),
            "roofline": {"bound": "hbm", "achieved": sw_gbs, "peak": peak, "unit": "GB/s",
                         "frac": sw_gbs / peak, "frac_of_nominal_8TBps": sw_gbs / 8000.0,
                         "traffic": _ncu_traffic(cfg, info),
                         "traffic_source": "profiles/ncu_switch_traffic.json (dram__bytes_read.sum + "
                                           "dram__bytes_write.sum of one ncu --set full capture of the same "
                                           "kernel on an identical-tile slice of the model, per layer x layers)",
                         "kernel": SWITCH_KERNELS.get(info.get("switch_kernel"), "switch_simt_kernel")
                                   + " (fused Eq. 10 switch)",
                         "peak_source": peak_src,
                         "bytes_per_launch": tb["switch"]},
            "cpu_baseline": cpu,
            "e2e": {"value": tok_bytes_all / e2e_s / 1e9, "unit": "GB/s", "ms_per_step": e2e_s * 1e3,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "lsw_decode_token_host"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sw.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="llama2-7b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--switch-impl", default="auto", choices=["auto", "tc", "simt"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-restore", action="store_true", help="skip the restore-from-pristine timing "
                    "(it needs one extra copy of the weights)")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="oracle seconds per reference-arm step (cpu_baseline uses max(this, 10))")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    import synth
    cfg = synth.get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
