"""The TP all-reduce call site executed on GPUs (-m gpu).

* One GPU: a tp_size = 1 ctx with a 1-rank NCCL communicator runs
  ncclAllReduce after every row-parallel (o, down) GEMV -- the identity, so
  the token's outputs must equal those of a ctx without a communicator bit
  for bit -- eagerly and replayed from a CUDA graph that captured the
  all-reduces (stream ordering, in-place use, capture); likewise the
  unmerged decode's and the prefill's all-reduce call sites.
* Two or more GPUs: scripts/tp_check.py under torchrun, every rank through
  lsw_attach_nccl + lsw_decode_token, compared with the oracle's full y and
  W slices.  Skipped when fewer than 2 GPUs are visible, so a multi-GPU box
  runs it unchanged.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if torch.cuda.is_available():
    from paper_2405_17741_b200 import harness as H
    from paper_2405_17741_b200.binding import LoraSwitch, nccl_version


@pytest.mark.parametrize("name", ["mini", "toy"])
def test_one_rank_allreduce_is_identity_eager_and_graph(name):
    cfg = synth.get_config(name)
    v, path = nccl_version()
    major, minor, patch = torch.cuda.nccl.version()
    assert v == major * 10000 + minor * 100 + patch, (v, path)
    outs = []
    for with_comm in (False, True):
        W, A, B, router = H.build_weights(cfg, "cuda")
        sw = H.make_switch(cfg, W, A, B, router)
        if with_comm:
            sw.attach_nccl(LoraSwitch.nccl_unique_id())
        info = sw.info()
        X1 = synth.gen_x1(cfg, 3, "cuda")
        xs = H.pack_xs(cfg, synth.gen_xs(cfg, "cuda"))
        ys = torch.empty(info["ys_elems"], dtype=torch.float32, device="cuda")
        idx = torch.empty(cfg.top_k, dtype=torch.int32, device="cuda")
        gate = torch.empty(cfg.top_k, dtype=torch.float32, device="cuda")
        res = []
        for t in range(2):
            sw.decode_token(X1[t], xs, ys, idx, gate)
            torch.cuda.synchronize()
            res.append(ys.clone())
        # the GEMVs (with their all-reduces) captured once, replayed
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        ys2 = torch.full_like(ys, float("nan"))
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            sw.decode_all_layers(xs, ys2, s)
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        res.append(ys2.clone())
        assert torch.equal(ys2, res[-2])               # same weights as token 2
        # the unmerged decode and prefill call sites too (all-reduce after o / down)
        sw.unmerge_all_layers()
        sw.router_topk(X1[2], idx, gate)
        sw.decode_all_layers_unmerged(xs, ys, idx, gate)
        torch.cuda.synchronize()
        res.append(ys.clone())
        if cfg.dtype == "bf16":
            T = 5
            gi = 3                                      # down: row-parallel
            d_in = cfg.kind_shape("down")[1]
            X = torch.randn(T, d_in, generator=torch.Generator().manual_seed(7)).to(torch.bfloat16).cuda()
            Y = torch.empty(T, cfg.kind_shape("down")[0], device="cuda")
            sw.prefill_group(0, gi, X, idx.repeat(T, 1), gate.repeat(T, 1), Y)
            torch.cuda.synchronize()
            res.append(Y.clone())
        assert sw.device_status() == 0
        outs.append(res)
        sw.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,name", [(2, "mini"), (2, "mini-r32"), (4, "mini")])
def test_tp_decode_through_nccl_matches_oracle(world, name):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "scripts", "tp_check.py"), "--config", name, "--tokens", "3"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and lines, (res.stdout[-2000:], res.stderr[-4000:])
    out = json.loads(lines[-1])
    assert out["ok"] and out["world"] == world, out
