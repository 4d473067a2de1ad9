"""ctypes binding of the C ABI in ``include/fsa_b200.h`` (``libfsa_b200.so``).

There is no fallback: if the shared object is missing or fails to load, every operator raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ._build import LIB_PATH

# fsa_status / fsa_dtype / fsa_op / device error bits — keep in sync with include/fsa_b200.h
FSA_OK, FSA_ERR_ARG, FSA_ERR_DTYPE, FSA_ERR_WORKSPACE, FSA_ERR_CUDA, FSA_ERR_ALIGN = range(6)
FSA_F32, FSA_F64, FSA_BF16, FSA_F16 = range(4)
FSA_OP_FWD1, FSA_OP_FWD2, FSA_OP_BWD1, FSA_OP_BWD2 = 1, 2, 3, 4
FSA_BWD_PLAN, FSA_BWD_TERMS, FSA_BWD_ROWS, FSA_BWD_APPLY, FSA_BWD_ALL = 1, 2, 4, 6, 7
FSA_FWD_SAMPLE, FSA_FWD_GATHER, FSA_FWD_ALL = 1, 2, 3
FSA_DEVERR_SEED_RANGE, FSA_DEVERR_INDEX_RANGE, FSA_DEVERR_NEG_TAKE = 1, 2, 4

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
_int = C.c_int
_sz = C.c_size_t

# name -> (restype, argtypes); exactly the symbols include/fsa_b200.h declares
SIGNATURES = {
    "fsa_version": (C.c_char_p, []),
    "fsa_status_string": (C.c_char_p, [_int]),
    "fsa_last_cuda_error": (_int, []),
    "fsa_set_device": (_int, [_int]),
    "fsa_launch_count": (C.c_ulonglong, []),
    "fsa_profile": (_int, [_int]),
    "fsa_profile_read": (_int, [_int, _p, _p, _p, C.POINTER(_int)]),
    "fsa_trace": (_int, [_p]),
    "fsa_trace_geometry": (_int, [C.POINTER(_int), C.POINTER(_int)]),
    "fsa_ws_bytes": (_sz, [_int, _i64, _i32, _i32, _i64, _int, _i64]),
    "fsa_read_error": (_int, [_p, _int, C.POINTER(_int), _p]),
    "fsa_fused_1hop_fwd": (_int, [_p, _p, _i64, _p, _i64, _i64, _int, _p, _i64, _i64, _i32, _u64, _int,
                                  _p, _p, _p, _i64, _p, _sz, _p]),
    "fsa_fused_2hop_fwd": (_int, [_p, _p, _i64, _p, _i64, _i64, _int, _p, _i64, _i64, _i32, _i32, _u64,
                                  _int, _p, _p, _p, _p, _p, _i64, _p, _sz, _p]),
    "fsa_fused_1hop_fwd_dseed": (_int, [_p, _p, _i64, _p, _i64, _i64, _int, _p, _i64, _i64, _i32, _p, _int,
                                        _p, _p, _p, _i64, _p, _sz, _p]),
    "fsa_fused_2hop_fwd_dseed": (_int, [_p, _p, _i64, _p, _i64, _i64, _int, _p, _i64, _i64, _i32, _i32, _p,
                                        _int, _p, _p, _p, _p, _p, _i64, _p, _sz, _p]),
    "fsa_fused_1hop_bwd": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i64, _p, _int, _p, _p, _p,
                                  _p, _sz, _p]),
    "fsa_fused_2hop_bwd": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i32, _i64, _p, _int, _p,
                                  _p, _p, _p, _sz, _p]),
    "fsa_fused_2hop_fwd_phase": (_int, [_p, _p, _i64, _p, _i64, _i64, _int, _p, _i64, _i64, _i32, _i32, _u64,
                                        _p, _int, _p, _p, _p, _p, _p, _i64, _p, _sz, _p, _int]),
    "fsa_fused_1hop_bwd_phase": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i64, _p, _int, _p, _p, _p,
                                        _p, _sz, _p, _int]),
    "fsa_fused_2hop_bwd_phase": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i32, _i64, _p, _int, _p,
                                        _p, _p, _p, _sz, _p, _int]),
    "fsa_zero_rows": (_int, [_p, _i64, _int, _p, _i64, _p]),
    "fsa_adamw_ws_bytes": (_sz, []),
    "fsa_adamw_step": (_int, [_int, _p, _p, _p, _p, _p, _p, C.c_double, C.c_double, C.c_double, C.c_double,
                              C.c_double, _p, _p, _sz, _p]),
    "fsa_sage_head_ws_bytes": (_sz, [_i64, _i32, _i32, _i32]),
    "fsa_sage_head_smem_bytes": (_sz, [_i32, _i32, _i32]),
    "fsa_sage_head_rows": (_int, [_p, _i64, _p, _p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _p, _i64,
                                  _p, _sz, _p]),
    "fsa_zero_rows_strided": (_int, [_p, _i64, _i64, _i64, _int, _p, _i64, _p]),
    "fsa_fused_2hop_bwd_phase_rows": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i32, _i64, _p, _i64, _i64,
                                             _int, _p, _sz, _p, _int]),
    "fsa_derive_states": (_int, [_p, _p, _p, _p, _i64, _p, _p]),
    "fsa_xorshift_steps": (_int, [_u64, _i64, _p, _p]),
    "fsa_jump": (_int, [_p, _p, _i64, _p, _p]),
    "fsa_umod": (_int, [_p, _p, _i64, _p, _p]),
    "fsa_div_check": (_int, [_int, _p, _p]),
    "fsa_bench_draws": (_int, [_int, _int, C.c_uint32, _int, _int, _p, _p]),
    "fsa_tune": (_int, [_int, _int]),
    "fsa_gather_rows": (_int, [_p, _i64, _i64, _int, _p, _i64, _p, _i64, _p]),
    "fsa_group_mean": (_int, [_p, _i64, _int, _p, _p, _i32, _i64, _i64, _int, _p, _i64, _int, _p]),
    "fsa_baseline_1hop_bwd": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i64, _p, _int, _p, _i64, _p, _sz, _p]),
    "fsa_baseline_2hop_bwd": (_int, [_p, _i64, _i64, _i64, _int, _p, _p, _i32, _i32, _i64, _p, _int, _p, _i64, _p,
                                      _sz, _p]),
}

_LIB = None


class FsaError(RuntimeError):
    """A C ABI call returned a non-OK status."""


def lib_path() -> Path:
    return LIB_PATH


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    # FSA_LIB: an alternative build of the same ABI (A/B experiments, instrumented builds)
    p = Path(path) if path is not None else Path(os.environ.get("FSA_LIB") or LIB_PATH)
    if not p.exists():
        raise ImportError(
            f"{p} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the FuseSampleAgg operator has no CPU fallback)"
        )
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(status: int, what: str) -> None:
    if status != FSA_OK:
        lib = load()
        msg = lib.fsa_status_string(status).decode()
        if status == FSA_ERR_CUDA:
            msg += f" (cudaError {lib.fsa_last_cuda_error()})"
        raise FsaError(f"{what}: {msg}")


def launch_count() -> int:
    """Kernels launched by libfsa_b200 in this process."""
    return int(load().fsa_launch_count())


def profile(enable: bool) -> None:
    check(load().fsa_profile(int(bool(enable))), "fsa_profile")


def profile_read(max_kernels: int = 64) -> dict:
    """{kernel name: (total device ms, launches)} recorded since profile(True)."""
    names = C.create_string_buffer(48 * max_kernels)
    ms = (C.c_double * max_kernels)()
    cnt = (C.c_int64 * max_kernels)()
    n = _int(0)
    check(load().fsa_profile_read(max_kernels, names, ms, cnt, C.byref(n)), "fsa_profile_read")
    out = {}
    raw = names.raw
    for i in range(n.value):
        nm = raw[48 * i:48 * (i + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (ms[i], int(cnt[i]))
    return out
