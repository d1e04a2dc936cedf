"""Seeded synthetic inputs for the LoRA-Switch hot path.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_2405_17741_b200/``).  It holds model geometry and seeded random
generators -- none of the method's arithmetic (no router, no merge, no GEMV).

Recipe:

* W  (backbone weight, one per adapted linear)  ~ N(0, 0.02^2), rounded (RNE) to
  the storage dtype by torch's own cast.  Llama init scale.
* A  (LoRA_DOWN, r x d_in, "W_down")       ~ U(-1/sqrt(d_in), +1/sqrt(d_in))
  (PEFT Kaiming-uniform bound).
* B  (LoRA_UP,  d_out x r, "W_up")          ~ N(0, sigma_B^2) with
  sigma_B = rho*0.02*sqrt(k) / (lora_scale*sqrt(r)*sigma_A), rho = 0.25,
  sigma_A = 1/sqrt(3 d_in), so that std(Delta W) ~= rho * std(W).  A real LoRA
  initialises B = 0, which would make parity vacuous.
* W_g (router, N x d_model)                ~ N(0, 1/d_model) -> logits ~ N(0,1).
* x1_t (router input, one per token, P:223 R7)    ~ N(0, I).
* x_{l,m} (GEMV input per layer/site group)       ~ N(0, I).

Seeds: base 2405177410 + tensor index, indices enumerated kind-major, then
layer, then W/A/B; then W_g; then the x1 stream; then the GEMV inputs.
Tensor-parallel shards are slices of the SAME full tensors (``shard_*``).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import torch

BASE_SEED = 2405177410
RHO = 0.25
W_STD = 0.02

# Adapted linears of a Llama/Mistral block ("all linears"; P:374 lists
# q, k, v, o, gate, down, up).  Order is the ABI's kind order.
KINDS = ("q", "k", "v", "o", "gate", "up", "down")
ROW_PARALLEL = {"o", "down"}          # Megatron row split (d_in sharded)
# GEMV groups that share one input vector in a real decode step (R18).
GROUPS = (("q", "k", "v"), ("o",), ("gate", "up"), ("down",))


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_layers: int
    d_model: int
    d_ff: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    n_experts: int
    rank: int
    top_k: int
    alpha: float
    dtype: str            # "bf16" | "f32"  (storage dtype of W, A, B, x)

    def kind_shape(self, kind: str) -> Tuple[int, int]:
        """(d_out, d_in) of one adapted linear, nn.Linear layout (R16)."""
        q = self.n_heads * self.head_dim
        kv = self.n_kv_heads * self.head_dim
        return {
            "q": (q, self.d_model), "k": (kv, self.d_model), "v": (kv, self.d_model),
            "o": (self.d_model, q),
            "gate": (self.d_ff, self.d_model), "up": (self.d_ff, self.d_model),
            "down": (self.d_model, self.d_ff),
        }[kind]

    def local_shape(self, kind: str, tp_rank: int = 0, tp_size: int = 1) -> Tuple[int, int]:
        d_out, d_in = self.kind_shape(kind)
        if tp_size == 1:
            return d_out, d_in
        if kind in ROW_PARALLEL:
            return d_out, len(range(*shard_range(d_in, tp_rank, tp_size)))
        return len(range(*shard_range(d_out, tp_rank, tp_size))), d_in

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    @property
    def lora_scale_for_recipe(self) -> float:
        # Only used to size sigma_B of the synthetic recipe above.
        return self.alpha / self.rank

    def n_weight_elems(self, tp_size: int = 1) -> int:
        tot = 0
        for kd in KINDS:
            o, i = self.local_shape(kd, 0, tp_size)
            tot += o * i
        return tot * self.n_layers

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; alpha = 16 everywhere (R3).
CONFIGS: Dict[str, Config] = {
    # toy: 2 layers, hidden 64, 4 experts r=4, top-2, fp32 (d_ff=128, R19)
    "toy": Config("toy", 2, 64, 128, 1, 1, 64, 4, 4, 2, 16.0, "f32"),
    "llama2-7b": Config("llama2-7b", 32, 4096, 11008, 32, 32, 128, 8, 16, 2, 16.0, "bf16"),
    "mistral-7b": Config("mistral-7b", 32, 4096, 14336, 32, 8, 128, 8, 16, 2, 16.0, "bf16"),
    "llama2-13b": Config("llama2-13b", 40, 5120, 13824, 40, 40, 128, 8, 32, 2, 16.0, "bf16"),
    # Small bf16 parity cases (oracle finishes in seconds; several 128-row tiles,
    # ragged row tail 704 = 5.5*128, GQA-shaped k/v).  Not bench lines.
    "mini": Config("mini", 2, 256, 704, 2, 1, 128, 8, 16, 2, 16.0, "bf16"),
    "mini-r32": Config("mini-r32", 2, 256, 704, 2, 1, 128, 8, 32, 2, 16.0, "bf16"),
    "mini-r4k4": Config("mini-r4k4", 2, 256, 704, 2, 1, 128, 16, 4, 4, 16.0, "bf16"),
    "mini-r64k3": Config("mini-r64k3", 1, 256, 704, 2, 1, 128, 4, 64, 3, 16.0, "bf16"),
    "mini-r48": Config("mini-r48", 1, 256, 704, 2, 1, 128, 4, 48, 2, 16.0, "bf16"),
    "mini-r64k4": Config("mini-r64k4", 1, 256, 704, 2, 1, 128, 8, 64, 4, 16.0, "bf16"),
    "mini-kN": Config("mini-kN", 1, 256, 704, 2, 1, 128, 4, 16, 4, 16.0, "bf16"),
    "mini-N64": Config("mini-N64", 1, 256, 704, 2, 1, 128, 64, 4, 2, 16.0, "bf16"),
    "mini-k1": Config("mini-k1", 2, 256, 704, 2, 1, 128, 4, 8, 1, 16.0, "bf16"),
    # Full router widths of configs[1..3] (d_model 4096 / 5120) on one thin layer:
    # GPU router parity at the real reduction length.
    "wide-d4096": Config("wide-d4096", 1, 4096, 128, 1, 1, 128, 8, 16, 2, 16.0, "bf16"),
    "wide-d5120": Config("wide-d5120", 1, 5120, 128, 1, 1, 128, 8, 32, 2, 16.0, "bf16"),
}


def sweep_configs() -> List[Config]:
    """configs[4]: rank 4..64 x top-k 1..4 x experts 4..16 on the 7B shape."""
    base = CONFIGS["llama2-7b"]
    out = []
    for n in (4, 8, 16):
        for r in (4, 8, 16, 32, 64):
            for k in (1, 2, 3, 4):
                if k <= n:
                    out.append(base.with_(name=f"sweep-n{n}-r{r}-k{k}", n_experts=n, rank=r, top_k=k))
    return out


def get_config(name: str) -> Config:
    if name in CONFIGS:
        return CONFIGS[name]
    for c in sweep_configs():
        if c.name == name:
            return c
    raise KeyError(name)


def shard_range(n: int, rank: int, size: int) -> Tuple[int, int]:
    """Contiguous, as-even-as-possible split of range(n) (first ranks get +1)."""
    base, rem = divmod(n, size)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


# ----------------------------------------------------------------------------
# Seeds
# ----------------------------------------------------------------------------

def _tensor_index(cfg: Config, kind: str, layer: int, which: str) -> int:
    return (KINDS.index(kind) * cfg.n_layers + layer) * 3 + "WAB".index(which)


def seed_of(cfg: Config, kind: str, layer: int, which: str) -> int:
    return BASE_SEED + _tensor_index(cfg, kind, layer, which)


def _seed_router(cfg: Config) -> int:
    return BASE_SEED + len(KINDS) * cfg.n_layers * 3


def _seed_x1(cfg: Config) -> int:
    return _seed_router(cfg) + 1


def _seed_xs(cfg: Config) -> int:
    return _seed_router(cfg) + 2


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


# ----------------------------------------------------------------------------
# Generators (full, unsharded tensors; shard with shard_* below)
# ----------------------------------------------------------------------------

def gen_W(cfg: Config, kind: str, layer: int, device="cpu") -> torch.Tensor:
    d_out, d_in = cfg.kind_shape(kind)
    g = _gen(seed_of(cfg, kind, layer, "W"), device)
    w = torch.randn(d_out, d_in, generator=g, device=device, dtype=torch.float32)
    w.mul_(W_STD)
    return w.to(cfg.torch_dtype)


def gen_A(cfg: Config, kind: str, layer: int, device="cpu") -> torch.Tensor:
    """LoRA_DOWN bank of one (kind, layer): [N, r, d_in]."""
    _, d_in = cfg.kind_shape(kind)
    g = _gen(seed_of(cfg, kind, layer, "A"), device)
    bound = 1.0 / math.sqrt(d_in)
    a = torch.rand(cfg.n_experts, cfg.rank, d_in, generator=g, device=device, dtype=torch.float32)
    a.mul_(2 * bound).sub_(bound)
    return a.to(cfg.torch_dtype)


def sigma_B(cfg: Config, kind: str) -> float:
    _, d_in = cfg.kind_shape(kind)
    sigma_a = 1.0 / math.sqrt(3 * d_in)
    return RHO * W_STD * math.sqrt(cfg.top_k) / (cfg.lora_scale_for_recipe * math.sqrt(cfg.rank) * sigma_a)


def gen_B(cfg: Config, kind: str, layer: int, device="cpu") -> torch.Tensor:
    """LoRA_UP bank of one (kind, layer): [N, d_out, r]."""
    d_out, _ = cfg.kind_shape(kind)
    g = _gen(seed_of(cfg, kind, layer, "B"), device)
    b = torch.randn(cfg.n_experts, d_out, cfg.rank, generator=g, device=device, dtype=torch.float32)
    b.mul_(sigma_B(cfg, kind))
    return b.to(cfg.torch_dtype)


def gen_router(cfg: Config, device="cpu") -> torch.Tensor:
    """W_g: [N, d_model]."""
    g = _gen(_seed_router(cfg), device)
    w = torch.randn(cfg.n_experts, cfg.d_model, generator=g, device=device, dtype=torch.float32)
    w.mul_(1.0 / math.sqrt(cfg.d_model))
    return w.to(cfg.torch_dtype)


def gen_x1(cfg: Config, n_tokens: int, device="cpu") -> torch.Tensor:
    """Router inputs x^1_t for t = 0..n_tokens-1: [T, d_model]."""
    g = _gen(_seed_x1(cfg), device)
    return torch.randn(n_tokens, cfg.d_model, generator=g, device=device, dtype=torch.float32).to(cfg.torch_dtype)


def gen_xs(cfg: Config, device="cpu") -> Dict[Tuple[int, int], torch.Tensor]:
    """GEMV inputs, one per (layer, group) -- full (unsharded) length d_in."""
    g = _gen(_seed_xs(cfg), device)
    out = {}
    for layer in range(cfg.n_layers):
        for gi, grp in enumerate(GROUPS):
            _, d_in = cfg.kind_shape(grp[0])
            out[(layer, gi)] = torch.randn(d_in, generator=g, device=device,
                                           dtype=torch.float32).to(cfg.torch_dtype)
    return out


# ----------------------------------------------------------------------------
# Tensor-parallel slicing: shards are slices of the full tensors.
# ----------------------------------------------------------------------------

def shard_W(cfg: Config, kind: str, W: torch.Tensor, rank: int, size: int) -> torch.Tensor:
    if size == 1:
        return W
    if kind in ROW_PARALLEL:
        s, e = shard_range(W.shape[-1], rank, size)
        return W[..., s:e]
    s, e = shard_range(W.shape[-2], rank, size)
    return W[..., s:e, :]


def shard_A(cfg: Config, kind: str, A: torch.Tensor, rank: int, size: int) -> torch.Tensor:
    """A [.., N, r, d_in]: columns sharded for row-parallel kinds, else replicated."""
    if size == 1 or kind not in ROW_PARALLEL:
        return A
    s, e = shard_range(A.shape[-1], rank, size)
    return A[..., s:e]


def shard_B(cfg: Config, kind: str, B: torch.Tensor, rank: int, size: int) -> torch.Tensor:
    """B [.., N, d_out, r]: rows sharded for column-parallel kinds, else replicated."""
    if size == 1 or kind in ROW_PARALLEL:
        return B
    s, e = shard_range(B.shape[-2], rank, size)
    return B[..., s:e, :]


def shard_x(cfg: Config, group_idx: int, x: torch.Tensor, rank: int, size: int) -> torch.Tensor:
    """GEMV input of a group: row-parallel groups take their d_in slice."""
    if size == 1 or GROUPS[group_idx][0] not in ROW_PARALLEL:
        return x
    s, e = shard_range(x.shape[-1], rank, size)
    return x[..., s:e]


def to_f64_numpy(t: torch.Tensor):
    """Exact widening of a storage-dtype tensor to a float64 numpy array."""
    return t.detach().to("cpu").to(torch.float64).numpy()


def dyadic(shape, lo: int, hi: int, denom: int, seed: int):
    """Integers in [lo, hi] divided by ``denom`` (a power of two): exact in any
    binary float format that holds the numerator; used for exact identities."""
    g = torch.Generator().manual_seed(seed)
    return (torch.randint(lo, hi + 1, tuple(shape), generator=g).to(torch.float64) / denom).numpy()
