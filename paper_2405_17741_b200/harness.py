"""Host-side setup: allocate the stacked per-kind tensors a ctx borrows and fill
them from the seeded generators in ``synth`` (device-side generation), plus
the token I/O packing used by lsw_decode_token.  No hot-path arithmetic here.
"""
from __future__ import annotations

from typing import Dict, Tuple

import torch

import synth

from .binding import LoraSwitch


def build_weights(cfg: synth.Config, device="cuda", tp_rank: int = 0, tp_size: int = 1,
                  kinds=synth.KINDS) -> Tuple[Dict[str, torch.Tensor], Dict[str, torch.Tensor],
                                               Dict[str, torch.Tensor], torch.Tensor]:
    """W[kind] [L, d_out, d_in], A[kind] [L, N, r, d_in], B[kind] [L, N, d_out, r]
    (this rank's shards, slices of the same full seeded tensors), router [N, d_model]."""
    W, A, B = {}, {}, {}
    dt = cfg.torch_dtype
    for kd in kinds:
        d_out, d_in = cfg.local_shape(kd, tp_rank, tp_size)
        W[kd] = torch.empty(cfg.n_layers, d_out, d_in, dtype=dt, device=device)
        A[kd] = torch.empty(cfg.n_layers, cfg.n_experts, cfg.rank, d_in, dtype=dt, device=device)
        B[kd] = torch.empty(cfg.n_layers, cfg.n_experts, d_out, cfg.rank, dtype=dt, device=device)
        for l in range(cfg.n_layers):
            W[kd][l].copy_(synth.shard_W(cfg, kd, synth.gen_W(cfg, kd, l, device), tp_rank, tp_size))
            A[kd][l].copy_(synth.shard_A(cfg, kd, synth.gen_A(cfg, kd, l, device), tp_rank, tp_size))
            B[kd][l].copy_(synth.shard_B(cfg, kd, synth.gen_B(cfg, kd, l, device), tp_rank, tp_size))
    router = synth.gen_router(cfg, device).contiguous()
    return W, A, B, router


def make_switch(cfg: synth.Config, W, A, B, router, impl: str = "auto", tp_rank: int = 0,
                tp_size: int = 1) -> LoraSwitch:
    return LoraSwitch(W, A, B, router, top_k=cfg.top_k, alpha=cfg.alpha, impl=impl,
                      tp_rank=tp_rank, tp_size=tp_size, row_parallel=tuple(synth.ROW_PARALLEL))


def pack_xs(cfg: synth.Config, xs: Dict[Tuple[int, int], torch.Tensor], tp_rank: int = 0,
            tp_size: int = 1) -> torch.Tensor:
    """Token GEMV inputs in lsw_decode_token order: layer-major, group-minor."""
    parts = []
    for l in range(cfg.n_layers):
        for gi in range(len(synth.GROUPS)):
            parts.append(synth.shard_x(cfg, gi, xs[(l, gi)], tp_rank, tp_size).reshape(-1))
    return torch.cat(parts).contiguous()


def ys_layout(cfg: synth.Config, tp_rank: int = 0, tp_size: int = 1):
    """[(layer, kind, offset, length)] of lsw_decode_token's packed output."""
    out, off = [], 0
    for l in range(cfg.n_layers):
        for grp in synth.GROUPS:
            for kd in grp:
                n = cfg.local_shape(kd, tp_rank, tp_size)[0]
                out.append((l, kd, off, n))
                off += n
    return out, off


def token_bytes(cfg: synth.Config, tp_size: int = 1) -> Dict[str, float]:
    """Algorithmic HBM bytes of one token per GPU (SURVEY d.3).

    switch: 2*s per W element (read + write) + s*K*(d_out + d_in) per matrix for
    the selected B/A slices, K = (#terms)*r with #terms = 2k (the Eq. 9/10
    concatenation; compaction may read fewer); merge/unmerge: K = k*r.
    gemv: s per W element + s*d_in + 4*d_out.  router: s*N*d_model + s*d_model.
    """
    s = cfg.elem_bytes
    w = sw = mg = gv = um = 0
    for kd in synth.KINDS:
        d_out, d_in = cfg.local_shape(kd, 0, tp_size)
        n = d_out * d_in * cfg.n_layers
        w += n
        sw += 2 * s * n + s * (2 * cfg.top_k * cfg.rank) * (d_out + d_in) * cfg.n_layers
        mg += 2 * s * n + s * (cfg.top_k * cfg.rank) * (d_out + d_in) * cfg.n_layers
        gv += s * n + (s * d_in + 4 * d_out) * cfg.n_layers
        # unmerged decode (Eq. 2): the GEMV's bytes + the k selected A and B slices
        um += s * n + (s * d_in + 4 * d_out) * cfg.n_layers + s * (cfg.top_k * cfg.rank) * (d_out + d_in) * cfg.n_layers
    rt = s * cfg.n_experts * cfg.d_model + s * cfg.d_model
    return {"w_elems": w, "switch": sw, "merge": mg, "gemv": gv, "router": rt,
            "token": sw + gv + rt, "unmerged_token": um + rt}


def token_flops(cfg: synth.Config, tp_size: int = 1, terms: int = None) -> float:
    """2*K*d_out*d_in per matrix for the switch contraction (K = terms*r)."""
    terms = 2 * cfg.top_k if terms is None else terms
    f = 0
    for kd in synth.KINDS:
        d_out, d_in = cfg.local_shape(kd, 0, tp_size)
        f += 2 * terms * cfg.rank * d_out * d_in * cfg.n_layers
    return float(f)
