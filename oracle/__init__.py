"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/liboracle.so (built from oracle/oracle.c).  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference legs) may import
this package.  It never imports paper_2008_11849_b200 and the CUDA path never imports it.

Every function takes float64 numpy arrays: callers widen the exact fp32/fp16 values the
GPU consumes (for fp16 cases W and X are the fp16-rounded values) before calling, so the
oracle sees bit-identical inputs.  See oracle/oracle.c for the paper
citations of each function.  Parity status: all functions pinned (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ORACLE_CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *ORACLE_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        lib.ref_to_dense_f64.argtypes = [i32, i32, P, P, P, P]
        lib.ref_to_dense_f64.restype = None
        lib.ref_gemm_f64.argtypes = [i32, i32, i64, P, i64, P, i64, P, i64, i32]
        lib.ref_gemm_f64.restype = None
        lib.ref_spmm_f64.argtypes = [i32, i32, i64, P, P, P, P, i64, P, i64, i32]
        lib.ref_spmm_f64.restype = ctypes.c_int
        lib.ref_im2col_f64.argtypes = [i32, i32, i32, i32, P, P]
        lib.ref_im2col_f64.restype = None
        lib.ref_conv3x3_f64.argtypes = [i32, i32, i32, i32, i32, P, P, P, P, P, i32]
        lib.ref_conv3x3_f64.restype = ctypes.c_int
        lib.ref_rel_l2.argtypes = [P, P, i64]
        lib.ref_rel_l2.restype = ctypes.c_double
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def to_dense(M, K, row_ptr, col_idx, val) -> np.ndarray:
    lib = _load()
    rp, ci, v = _c(row_ptr, np.int32), _c(col_idx, np.int32), _c(val, np.float64)
    out = np.empty((M, K), np.float64)
    lib.ref_to_dense_f64(M, K, _p(rp), _p(ci), _p(v), _p(out))
    return out


def gemm(A: np.ndarray, B: np.ndarray, threads: int | None = None) -> np.ndarray:
    lib = _load()
    A, B = _c(A, np.float64), _c(B, np.float64)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N), np.float64)
    lib.ref_gemm_f64(M, K, N, _p(A), K, _p(B), N, _p(C), N, threads or default_threads())
    return C


def spmm(M, K, row_ptr, col_idx, val, X: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Y (M x N) = to_dense(W) @ X, X is (K x N) float64 (N = X.shape[1])."""
    lib = _load()
    rp, ci, v = _c(row_ptr, np.int32), _c(col_idx, np.int32), _c(val, np.float64)
    X = _c(X, np.float64)
    assert X.shape[0] == K
    N = X.shape[1]
    Y = np.empty((M, N), np.float64)
    rc = lib.ref_spmm_f64(M, K, N, _p(rp), _p(ci), _p(v), _p(X), N, _p(Y), N,
                          threads or default_threads())
    if rc != 0:
        raise MemoryError("ref_spmm_f64 failed")
    return Y


def im2col(x: np.ndarray) -> np.ndarray:
    """x [C_in][B][H][W] -> (9*C_in) x (B*H*W)."""
    lib = _load()
    x = _c(x, np.float64)
    C, B, H, W = x.shape
    cols = np.empty((9 * C, B * H * W), np.float64)
    lib.ref_im2col_f64(C, B, H, W, _p(x), _p(cols))
    return cols


def conv3x3(C_out, row_ptr, col_idx, val, x: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Direct 3x3 conv, pad 1, stride 1; W CSR (C_out x 9*C_in); x [C_in][B][H][W]."""
    lib = _load()
    x = _c(x, np.float64)
    C_in, B, H, W = x.shape
    rp, ci, v = _c(row_ptr, np.int32), _c(col_idx, np.int32), _c(val, np.float64)
    y = np.empty((C_out, B, H, W), np.float64)
    rc = lib.ref_conv3x3_f64(C_out, C_in, B, H, W, _p(rp), _p(ci), _p(v), _p(x), _p(y),
                             threads or default_threads())
    if rc != 0:
        raise MemoryError("ref_conv3x3_f64 failed")
    return y


def rel_l2(a: np.ndarray, ref: np.ndarray) -> float:
    lib = _load()
    a, ref = _c(a, np.float64).reshape(-1), _c(ref, np.float64).reshape(-1)
    assert a.size == ref.size
    return float(lib.ref_rel_l2(_p(a), _p(ref), a.size))
