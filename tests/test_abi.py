"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/lsw.h declares; host-side validation errors need no GPU (-m "not gpu")."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = ""
    for name in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if name.endswith(".h"):
            with open(os.path.join(ROOT, "include", name)) as f:
                src += f.read()
    return sorted(set(re.findall(r"^LSW_API\s+[\w\s\*]+?\b(lsw_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2405_17741_b200 as L
    return L


def test_header_declares_the_four_boundary_calls():
    syms = _declared_symbols()
    for s in ("lsw_router_topk", "lsw_merge_all_layers", "lsw_unmerge_all_layers", "lsw_decode_linear"):
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    lib = ctypes.CDLL(L.LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(lib, s), s
    assert set(L.SYMBOLS) == set(syms)
    assert L.lib().lsw_abi_version() == 1


def _cfg(L, **kw):
    base = dict(n_layers=2, n_experts=4, rank=4, top_k=2, alpha=16.0, dtype=0, d_model=64,
                tp_rank=0, tp_size=1, impl=1)
    base.update(kw)
    return L.binding.Config(**base)


def _kinds(L, d_in=64, d_out=64):
    kinds = (L.binding.KindDesc * 7)()
    for i in range(7):
        kinds[i] = L.binding.KindDesc(W=4096, A=8192, B=16384, d_out=d_out, d_in=d_in, row_parallel=0)
    return kinds


@pytest.mark.parametrize("kw,status", [
    (dict(top_k=5), 2), (dict(top_k=0), 2), (dict(n_experts=65, top_k=2), 2), (dict(dtype=7), 1),
    (dict(tp_rank=2, tp_size=2), 1), (dict(impl=9), 1), (dict(rank=0), 2), (dict(d_model=60), 2),
    (dict(impl=2, dtype=0), 8),
])
def test_create_validation_errors_without_gpu(L, kw, status):
    h = ctypes.c_void_p()
    st = L.lib().lsw_create(ctypes.byref(_cfg(L, **kw)), _kinds(L), 1024, ctypes.byref(h))
    assert st == status, L.lib().lsw_last_error()
    assert h.value is None
    assert L.lib().lsw_last_error()


def test_create_shape_errors_name_the_shapes(L):
    h = ctypes.c_void_p()
    st = L.lib().lsw_create(ctypes.byref(_cfg(L)), _kinds(L, d_in=60), 1024, ctypes.byref(h))
    assert st == 2 and b"60" in L.lib().lsw_last_error()
    st = L.lib().lsw_create(None, _kinds(L), 1024, ctypes.byref(h))
    assert st == 1
    assert L.lib().lsw_router_topk(None, None, None, None, None) == 1
    assert L.lib().lsw_unmerge_all_layers(None, None) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2405_17741_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "lsw_oracle" not in src, f


def test_null_ctx_is_refused_by_every_entry_point(L):
    """Every hot call validates before it enqueues anything: a null ctx (or
    null argument) returns LSW_E_ARG on a CPU-only box, no CUDA call made."""
    lib = L.lib()
    E_ARG = 1
    assert lib.lsw_merge_all_layers(None, None, None, None) == E_ARG
    assert lib.lsw_restore_merge_all_layers(None, None, None, None) == E_ARG
    assert lib.lsw_decode_linear(None, 0, 0, None, None, None) == E_ARG
    assert lib.lsw_decode_group(None, 0, 0, None, None, None) == E_ARG
    assert lib.lsw_decode_all_layers(None, None, None, None) == E_ARG
    assert lib.lsw_decode_group_unmerged(None, 0, 0, None, None, None, None, None) == E_ARG
    assert lib.lsw_decode_all_layers_unmerged(None, None, None, None, None, None) == E_ARG
    assert lib.lsw_decode_token(None, None, None, None, None, None, None) == E_ARG
    assert lib.lsw_decode_token_fused(None, None, None, None, None, None, None) == E_ARG
    assert lib.lsw_decode_token_host(None, None, None, None, None, None, None) == E_ARG
    assert lib.lsw_prefill_group(None, 0, 0, None, 1, None, None, None, None) == E_ARG
    assert b"null" in lib.lsw_last_error()


def test_nccl_is_the_process_copy_torch_loaded(L):
    """liblsw does not link NCCL; its first NCCL call binds
    the libnccl.so.2 already in the process (torch's), so the TP all-reduce
    and torch.distributed share one NCCL.  Needs no GPU."""
    import torch
    v, path = L.binding.nccl_version()
    major, minor, patch = torch.cuda.nccl.version()
    assert v == major * 10000 + minor * 100 + patch, (v, path)
    maps = [ln.split()[-1] for ln in open("/proc/self/maps") if "libnccl" in ln]
    assert os.path.realpath(path) in {os.path.realpath(m) for m in maps}
    assert L.lib().lsw_nccl_version(None, None, 0) == 1
