"""Thin ctypes binding over liblsw.so (include/lsw.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  torch supplies device memory (tensors are passed by data_ptr),
streams (torch.cuda.current_stream()) and, for TP, the process group used to
broadcast the NCCL unique id.  If the library is missing this module raises at
import -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblsw.so")

KINDS = ("q", "k", "v", "o", "gate", "up", "down")
GROUPS = (("q", "k", "v"), ("o",), ("gate", "up"), ("down",))
MAX_TOPK = 8

LSW_OK = 0
STATUS = {0: "LSW_OK", 1: "LSW_E_ARG", 2: "LSW_E_SHAPE", 3: "LSW_E_STATE", 4: "LSW_E_CUDA",
          5: "LSW_E_NCCL", 6: "LSW_E_DEVICE", 7: "LSW_E_OOM", 8: "LSW_E_UNSUPPORTED"}
DTYPE = {torch.bfloat16: 1, torch.float32: 0}
IMPL = {"auto": 0, "simt": 1, "tc": 2}
IMPL_NAME = {v: k for k, v in IMPL.items()}

# Exported symbols the header declares (checked by tests/test_abi.py).
SYMBOLS = (
    "lsw_abi_version", "lsw_last_error", "lsw_create", "lsw_destroy", "lsw_get_info",
    "lsw_nccl_get_unique_id", "lsw_attach_nccl", "lsw_nccl_version", "lsw_router_topk", "lsw_merge_all_layers",
    "lsw_unmerge_all_layers", "lsw_attach_pristine", "lsw_restore_merge_all_layers", "lsw_decode_linear", "lsw_decode_group", "lsw_decode_all_layers",
    "lsw_decode_group_unmerged", "lsw_decode_all_layers_unmerged", "lsw_decode_token", "lsw_decode_token_fused",
    "lsw_decode_token_host", "lsw_device_status", "lsw_prefill_group",
    "lsw_debug_set_option", "lsw_debug_merge_per_matrix",   # include/lsw_debug.h
)


class LswError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class KindDesc(ctypes.Structure):
    _fields_ = [("W", ctypes.c_void_p), ("A", ctypes.c_void_p), ("B", ctypes.c_void_p),
                ("d_out", ctypes.c_int64), ("d_in", ctypes.c_int64),
                ("row_parallel", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_experts", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("alpha", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("d_model", ctypes.c_int64), ("tp_rank", ctypes.c_int32), ("tp_size", ctypes.c_int32),
                ("impl", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("tiles_total", ctypes.c_int64), ("switch_impl", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("tile_m", ctypes.c_int32), ("tile_n", ctypes.c_int32), ("merged", ctypes.c_int32),
                ("num_sms", ctypes.c_int32), ("kernel_launches", ctypes.c_uint64),
                ("packed_bytes", ctypes.c_int64), ("xs_elems", ctypes.c_int64), ("ys_elems", ctypes.c_int64),
                ("switch_kernel", ctypes.c_int32), ("reserved", ctypes.c_int32)]


def load_library(path: str = LIB_PATH, strict: bool = True) -> ctypes.CDLL:
    """strict=False (tuning scripts only: A/B against an older build) skips
    entry points the library does not export."""
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA library is required; there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "lsw_abi_version": (i32, []),
        "lsw_last_error": (ctypes.c_char_p, []),
        "lsw_create": (i32, [ctypes.POINTER(Config), ctypes.POINTER(KindDesc), vp, ctypes.POINTER(vp)]),
        "lsw_destroy": (i32, [vp]),
        "lsw_get_info": (i32, [vp, ctypes.POINTER(Info)]),
        "lsw_nccl_get_unique_id": (i32, [vp]),
        "lsw_attach_nccl": (i32, [vp, vp]),
        "lsw_nccl_version": (i32, [ctypes.POINTER(i32), ctypes.c_char_p, i64]),
        "lsw_router_topk": (i32, [vp, vp, vp, vp, vp]),
        "lsw_merge_all_layers": (i32, [vp, vp, vp, vp]),
        "lsw_unmerge_all_layers": (i32, [vp, vp]),
        "lsw_attach_pristine": (i32, [vp, ctypes.POINTER(vp)]),
        "lsw_restore_merge_all_layers": (i32, [vp, vp, vp, vp]),
        "lsw_decode_linear": (i32, [vp, i32, i32, vp, vp, vp]),
        "lsw_decode_group": (i32, [vp, i32, i32, vp, vp, vp]),
        "lsw_decode_all_layers": (i32, [vp, vp, vp, vp]),
        "lsw_decode_group_unmerged": (i32, [vp, i32, i32, vp, vp, vp, vp, vp]),
        "lsw_decode_all_layers_unmerged": (i32, [vp, vp, vp, vp, vp, vp]),
        "lsw_decode_token": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "lsw_decode_token_fused": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "lsw_decode_token_host": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "lsw_device_status": (i32, [vp, vp, ctypes.POINTER(i32)]),
        "lsw_prefill_group": (i32, [vp, i32, i32, vp, i64, vp, vp, vp, vp]),
        "lsw_debug_set_option": (i32, [ctypes.c_char_p, ctypes.c_char_p]),
        "lsw_debug_merge_per_matrix": (i32, [vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        if not strict and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB: Optional[ctypes.CDLL] = None


def set_option(key: Optional[str], value=None):
    """include/lsw_debug.h lsw_debug_set_option: variant / tuning options read
    at ctx creation (key None clears all, value None unsets)."""
    enc = lambda v: None if v is None else str(v).encode()
    _check(lib().lsw_debug_set_option(enc(key), enc(value)))


class options:
    """Context manager: set options for the ctxs created inside, then clear them."""

    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k in self.kv:
            set_option(k, None)


def nccl_version():
    """(NCCL_VERSION_CODE, file) of the libnccl.so.2 liblsw bound (lsw_nccl_version)."""
    v = ctypes.c_int32(0)
    buf = ctypes.create_string_buffer(4096)
    _check(lib().lsw_nccl_version(ctypes.byref(v), buf, len(buf)))
    return v.value, buf.value.decode()


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load_library()
    return _LIB


def _check(st: int):
    if st != LSW_OK:
        raise LswError(st, lib().lsw_last_error().decode(errors="replace"))


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class LoraSwitch:
    """One ctx of the C library.  Tensors stay owned by the caller (kept alive
    here by reference); W tensors are mutated in place by merge/unmerge.

    W[kind] [L, d_out, d_in], A[kind] [L, N, r, d_in], B[kind] [L, N, d_out, r],
    router_w [N, d_model]; all on the current CUDA device, same dtype.
    """

    def __init__(self, W: Dict[str, torch.Tensor], A: Dict[str, torch.Tensor], B: Dict[str, torch.Tensor],
                 router_w: torch.Tensor, *, top_k: int, alpha: float, impl: str = "auto",
                 tp_rank: int = 0, tp_size: int = 1, row_parallel: Sequence[str] = ("o", "down")):
        self._keep = (W, A, B, router_w)
        dt = router_w.dtype
        L, N, r, _ = A["q"].shape
        cfg = Config(n_layers=L, n_experts=N, rank=r, top_k=top_k, alpha=alpha, dtype=DTYPE[dt],
                     d_model=router_w.shape[1], tp_rank=tp_rank, tp_size=tp_size, impl=IMPL[impl])
        kinds = (KindDesc * 7)()
        for i, kd in enumerate(KINDS):
            for t in (W[kd], A[kd], B[kd]):
                if not t.is_contiguous() or t.dtype != dt or not t.is_cuda:
                    raise ValueError(f"kind {kd}: tensors must be contiguous CUDA {dt}")
            kinds[i] = KindDesc(W=W[kd].data_ptr(), A=A[kd].data_ptr(), B=B[kd].data_ptr(),
                                d_out=W[kd].shape[1], d_in=W[kd].shape[2],
                                row_parallel=int(kd in row_parallel))
        h = ctypes.c_void_p()
        _check(lib().lsw_create(ctypes.byref(cfg), kinds, router_w.data_ptr(), ctypes.byref(h)))
        self._h = h
        self.top_k = top_k
        self.dtype = dt
        self.d_model = router_w.shape[1]

    # --- lifecycle --------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().lsw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        inf = Info()
        _check(lib().lsw_get_info(self._h, ctypes.byref(inf)))
        d = {f: getattr(inf, f) for f, _ in Info._fields_}
        d["switch_impl"] = IMPL_NAME.get(d["switch_impl"], d["switch_impl"])
        return d

    def attach_nccl(self, unique_id: bytes):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib().lsw_attach_nccl(self._h, buf))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().lsw_nccl_get_unique_id(buf))
        return buf.raw

    # --- the four calls of the boundary -----------------------------------
    def router_topk(self, x1: torch.Tensor, idx: torch.Tensor, gate: torch.Tensor, stream=None):
        _check(lib().lsw_router_topk(self._h, _ptr(x1), _ptr(idx), _ptr(gate), _stream(stream)))

    def merge_all_layers(self, idx: torch.Tensor, gate: torch.Tensor, stream=None):
        _check(lib().lsw_merge_all_layers(self._h, _ptr(idx), _ptr(gate), _stream(stream)))

    def attach_pristine(self, P: Dict[str, torch.Tensor]):
        """Pristine copies of W (same shapes/dtype, device) for the restore switch."""
        for kd in KINDS:
            t = P[kd]
            if not t.is_contiguous() or t.dtype != self.dtype or not t.is_cuda:
                raise ValueError(f"pristine {kd}: must be a contiguous CUDA {self.dtype} tensor")
        self._keep_p = P
        arr = (ctypes.c_void_p * 7)(*[P[kd].data_ptr() for kd in KINDS])
        _check(lib().lsw_attach_pristine(self._h, arr))

    def restore_merge_all_layers(self, idx: torch.Tensor, gate: torch.Tensor, stream=None):
        """W <- RNE(P + Delta(idx, gate)) from the attached pristine copy, any state."""
        _check(lib().lsw_restore_merge_all_layers(self._h, _ptr(idx), _ptr(gate), _stream(stream)))

    def unmerge_all_layers(self, stream=None):
        _check(lib().lsw_unmerge_all_layers(self._h, _stream(stream)))

    def decode_linear(self, layer: int, kind: str, x: torch.Tensor, y: torch.Tensor, stream=None):
        _check(lib().lsw_decode_linear(self._h, layer, KINDS.index(kind), _ptr(x), _ptr(y), _stream(stream)))

    # --- conveniences built from the same kernels ---------------------------
    def decode_group(self, layer: int, group: int, x: torch.Tensor, y: torch.Tensor, stream=None):
        _check(lib().lsw_decode_group(self._h, layer, group, _ptr(x), _ptr(y), _stream(stream)))

    def decode_all_layers(self, xs, ys, stream=None):
        """Every group GEMV of every layer (packed xs -> packed ys), decoder order."""
        _check(lib().lsw_decode_all_layers(self._h, _ptr(xs), _ptr(ys), _stream(stream)))

    def decode_group_unmerged(self, layer: int, group: int, x, y, idx, gate, stream=None):
        """y = W x + sum_j (alpha/r) g_j B_j (A_j x) on the UN-merged weights (Eq. 2)."""
        _check(lib().lsw_decode_group_unmerged(self._h, layer, group, _ptr(x), _ptr(y), _ptr(idx), _ptr(gate),
                                               _stream(stream)))

    def prefill_group(self, layer: int, group: int, X, idx, gate, Y, stream=None):
        """Y[t] = W x_t + sum_j (alpha/r) g_tj B_j (A_j x_t) for T tokens with per-token decisions
        (X [T, d_in], idx [T, k] int32, gate [T, k] fp32, Y [T, rows] fp32; unmerged ctx)."""
        _check(lib().lsw_prefill_group(self._h, layer, group, _ptr(X), int(X.shape[0]), _ptr(idx), _ptr(gate),
                                       _ptr(Y), _stream(stream)))

    def decode_all_layers_unmerged(self, xs, ys, idx, gate, stream=None):
        _check(lib().lsw_decode_all_layers_unmerged(self._h, _ptr(xs), _ptr(ys), _ptr(idx), _ptr(gate),
                                                    _stream(stream)))

    def decode_token(self, x1, xs, ys, idx, gate, stream=None):
        _check(lib().lsw_decode_token(self._h, _ptr(x1), _ptr(xs), _ptr(ys), _ptr(idx), _ptr(gate),
                                      _stream(stream)))

    def decode_token_fused(self, x1, xs, ys, idx, gate, stream=None):
        """The token with the switch and the GEMVs fused in one launch (4 B/element)."""
        _check(lib().lsw_decode_token_fused(self._h, _ptr(x1), _ptr(xs), _ptr(ys), _ptr(idx), _ptr(gate),
                                            _stream(stream)))

    def decode_token_host(self, x1_h, xs_h, ys_h, idx_h, gate_h, stream=None):
        _check(lib().lsw_decode_token_host(self._h, _ptr(x1_h), _ptr(xs_h), _ptr(ys_h), _ptr(idx_h),
                                           _ptr(gate_h), _stream(stream)))

    def debug_merge_per_matrix(self, idx, gate, stream=None):
        """Launch-count ablation (include/lsw_debug.h): the merge as 7*L launches."""
        _check(lib().lsw_debug_merge_per_matrix(self._h, _ptr(idx), _ptr(gate), _stream(stream)))

    def device_status(self, stream=None) -> int:
        code = ctypes.c_int32(0)
        st = lib().lsw_device_status(self._h, _stream(stream), ctypes.byref(code))
        if st not in (LSW_OK, 6):
            _check(st)
        return code.value
