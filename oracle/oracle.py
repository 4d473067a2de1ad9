"""ctypes wrapper of the C restatement ``oracle/fsa_oracle.c`` — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) import this
module; it is the parity checker and the CPU baseline, never the product path.  Numpy in,
numpy out, same semantics as the reference ``fsa.kernels`` / ``fsa.fused`` functions it
restates (see the file:line citations in fsa_oracle.c).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "fsa_oracle.c"
LIB = HERE / "_build" / "libfsa_oracle.so"
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        LIB.parent.mkdir(parents=True, exist_ok=True)
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(["gcc", *CFLAGS, "-o", str(tmp), str(SRC)], check=True)
        os.replace(tmp, LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(LIB))
        u64, i64, p, i32 = C.c_uint64, C.c_int64, C.c_void_p, C.c_int
        lib.oracle_derive.restype = u64
        lib.oracle_derive.argtypes = [u64, u64, u64, u64]
        lib.oracle_splitmix64.restype = u64
        lib.oracle_splitmix64.argtypes = [u64]
        lib.oracle_xorshift_steps.argtypes = [u64, i64, p]
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_get_threads.restype = i32
        lib.oracle_sample_1hop.argtypes = [p, p, p, i64, i64, i64, u64, p, p]
        lib.oracle_sample_2hop.argtypes = [p, p, p, i64, i64, i64, i64, u64, p, p, p, p]
        for sfx in ("f32", "f64"):
            getattr(lib, f"oracle_fused_1hop_{sfx}").argtypes = [p, p, p, i64, p, i64, i64, i64, u64, i32, p, p, p]
            getattr(lib, f"oracle_fused_2hop_{sfx}").argtypes = [p, p, p, i64, p, i64, i64, i64, i64, u64, i32,
                                                                 p, p, p, p, p]
            getattr(lib, f"oracle_bwd_1hop_{sfx}").argtypes = [p, i64, i64, p, p, i64, i64, p]
            getattr(lib, f"oracle_bwd_1hop_{sfx}").restype = i32
            getattr(lib, f"oracle_bwd_2hop_{sfx}").argtypes = [p, i64, i64, p, p, i64, i64, i64, p]
            getattr(lib, f"oracle_bwd_2hop_{sfx}").restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _sfx(dtype) -> str:
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise ValueError(f"oracle supports float32/float64, got {dtype}")


def set_threads(n: int) -> None:
    load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(load().oracle_get_threads())


def derive_state(base: int, root: int, hop: int, index: int) -> int:
    M = (1 << 64) - 1
    return int(load().oracle_derive(base & M, root & M, hop & M, index & M))


def splitmix64(z: int) -> int:
    return int(load().oracle_splitmix64(z & ((1 << 64) - 1)))


def xorshift_steps(state: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    load().oracle_xorshift_steps(state, n, _ptr(out))
    return out


def _graph_arrays(rowptr, col):
    return np.ascontiguousarray(rowptr, dtype=np.int32), np.ascontiguousarray(col, dtype=np.int32)


def sample_1hop(rowptr, col, seeds, k, base_seed, root_offset=0):
    rp, cl = _graph_arrays(rowptr, col)
    s = np.ascontiguousarray(seeds, dtype=np.int64)
    B = len(s)
    samples = np.empty((B, k), np.int32)
    takes = np.empty(B, np.int32)
    load().oracle_sample_1hop(_ptr(rp), _ptr(cl), _ptr(s), B, root_offset, k, base_seed & ((1 << 64) - 1),
                              _ptr(samples), _ptr(takes))
    return samples, takes


def sample_2hop(rowptr, col, seeds, k1, k2, base_seed, root_offset=0):
    rp, cl = _graph_arrays(rowptr, col)
    s = np.ascontiguousarray(seeds, dtype=np.int64)
    B = len(s)
    s1 = np.empty((B, k1), np.int32)
    s2 = np.empty((B, k1, k2), np.int32)
    t1 = np.empty(B, np.int32)
    t2 = np.empty((B, k1), np.int32)
    load().oracle_sample_2hop(_ptr(rp), _ptr(cl), _ptr(s), B, root_offset, k1, k2, base_seed & ((1 << 64) - 1),
                              _ptr(s1), _ptr(s2), _ptr(t1), _ptr(t2))
    return s1, s2, t1, t2


def fused_1hop(rowptr, col, X, seeds, k, base_seed, save=True, root_offset=0):
    """kernels.fused_1hop: returns (out, samples, takes) (samples/takes None when not saved)."""
    rp, cl = _graph_arrays(rowptr, col)
    X = np.ascontiguousarray(X)
    s = np.ascontiguousarray(seeds, dtype=np.int64)
    B, D = len(s), X.shape[1]
    out = np.empty((B, D), X.dtype)
    samples = np.empty((B, k), np.int32) if save else None
    takes = np.empty(B, np.int32) if save else None
    getattr(load(), f"oracle_fused_1hop_{_sfx(X.dtype)}")(
        _ptr(rp), _ptr(cl), _ptr(X), D, _ptr(s), B, root_offset, k, base_seed & ((1 << 64) - 1), int(save),
        _ptr(samples) if save else None, _ptr(takes) if save else None, _ptr(out))
    return out, samples, takes


def fused_2hop(rowptr, col, X, seeds, k1, k2, base_seed, save=True, root_offset=0):
    """kernels.fused_2hop: returns (out, s1, s2, take1, take2)."""
    rp, cl = _graph_arrays(rowptr, col)
    X = np.ascontiguousarray(X)
    s = np.ascontiguousarray(seeds, dtype=np.int64)
    B, D = len(s), X.shape[1]
    out = np.empty((B, D), X.dtype)
    if save:
        s1 = np.empty((B, k1), np.int32)
        s2 = np.empty((B, k1, k2), np.int32)
        t1 = np.empty(B, np.int32)
        t2 = np.empty((B, k1), np.int32)
        ptrs = [_ptr(s1), _ptr(s2), _ptr(t1), _ptr(t2)]
    else:
        s1 = s2 = t1 = t2 = None
        ptrs = [None] * 4
    getattr(load(), f"oracle_fused_2hop_{_sfx(X.dtype)}")(
        _ptr(rp), _ptr(cl), _ptr(X), D, _ptr(s), B, root_offset, k1, k2, base_seed & ((1 << 64) - 1),
        int(save), *ptrs, _ptr(out))
    return out, s1, s2, t1, t2


def backward_1hop(grad_out, samples, takes, num_nodes, out=None):
    g = np.ascontiguousarray(grad_out)
    smp = np.ascontiguousarray(samples, dtype=np.int32)
    tk = np.ascontiguousarray(takes, dtype=np.int32)
    B, D = g.shape
    if out is None:
        out = np.empty((num_nodes, D), g.dtype)
    rc = getattr(load(), f"oracle_bwd_1hop_{_sfx(g.dtype)}")(_ptr(g), B, D, _ptr(smp), _ptr(tk),
                                                             smp.shape[1], num_nodes, _ptr(out))
    if rc:
        raise MemoryError("oracle backward allocation failed")
    return out


def backward_2hop(grad_out, s1, s2, num_nodes, out=None):
    g = np.ascontiguousarray(grad_out)
    a1 = np.ascontiguousarray(s1, dtype=np.int32)
    a2 = np.ascontiguousarray(s2, dtype=np.int32)
    B, D = g.shape
    if out is None:
        out = np.empty((num_nodes, D), g.dtype)
    rc = getattr(load(), f"oracle_bwd_2hop_{_sfx(g.dtype)}")(_ptr(g), B, D, _ptr(a1), _ptr(a2),
                                                             a1.shape[1], a2.shape[2], num_nodes, _ptr(out))
    if rc:
        raise MemoryError("oracle backward allocation failed")
    return out
