"""Thin ctypes binding of libsparsert.so (include/sparsert.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  PyTorch is used for device memory and streams (tensors are passed as raw
device pointers).  There is no CPU fallback: if the library is missing or fails to
load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SPARSERT_LIB: load an alternative build of the same library (A/B experiments, scripts/)
LIB_PATH = os.environ.get("SPARSERT_LIB") or os.path.join(_PKG, "libsparsert.so")

SPARSE_OK, SPARSE_EINVAL, SPARSE_EMATRIX, SPARSE_EUNSUPPORTED = 0, 1, 2, 3
SPARSE_ENOMEM, SPARSE_ECUDA, SPARSE_EINTERNAL = 4, 5, 6
SPARSE_F32, SPARSE_F16, SPARSE_BF16 = 0, 1, 2
SPARSE_SPMM, SPARSE_CONV3X3 = 0, 1
SPARSE_DEVICE_HOST_ONLY = -2

STATUS_NAMES = {0: "SPARSE_OK", 1: "SPARSE_EINVAL", 2: "SPARSE_EMATRIX", 3: "SPARSE_EUNSUPPORTED",
                4: "SPARSE_ENOMEM", 5: "SPARSE_ECUDA", 6: "SPARSE_EINTERNAL"}

# every symbol include/sparsert.h declares (checked by tests/test_capi_host.py)
EXPORTED = ["sparse_plan_opts_init", "sparse_plan_create", "sparse_spmm", "sparse_conv3x3",
            "sparse_spmm_ex", "sparse_conv3x3_ex", "sparse_linear", "sparse_conv1x1", "sparse_conv3x3_nhwc",
            "plan_destroy", "sparse_plan_destroy", "sparse_plan_info", "sparse_plan_dump",
            "sparse_last_error", "sparse_version"]


class SparseRTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class sparse_plan_opts(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("c_in", ctypes.c_int32), ("h", ctypes.c_int32),
                ("w", ctypes.c_int32), ("n_hint", ctypes.c_int64), ("tune", ctypes.c_int32),
                ("device", ctypes.c_int32), ("drop_zeros", ctypes.c_int32),
                ("warps", ctypes.c_int32), ("rows_per_warp", ctypes.c_int32),
                ("k_chunk", ctypes.c_int32), ("split_k", ctypes.c_int32),
                ("k_split", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("executor", ctypes.c_int32), ("jit_rows", ctypes.c_int32),
                ("jit_warps", ctypes.c_int32), ("x_multicast", ctypes.c_int32),
                ("x_source", ctypes.c_int32), ("conv_kernel", ctypes.c_int32),
                ("row_order", ctypes.c_int32), ("tc_min_density", ctypes.c_int32),
                ("plan_source", ctypes.c_int32), ("cta_pair", ctypes.c_int32)]


class sparse_epilogue(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_float), ("bias", ctypes.c_void_p), ("relu", ctypes.c_int32)]


class sparse_plan_info_t(ctypes.Structure):
    _fields_ = [("nnz", ctypes.c_int64), ("plan_bytes", ctypes.c_int64),
                ("M", ctypes.c_int32), ("K", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("panels", ctypes.c_int32), ("warps", ctypes.c_int32),
                ("rows_per_warp", ctypes.c_int32), ("cols_per_lane", ctypes.c_int32),
                ("n_tile", ctypes.c_int32), ("k_chunk", ctypes.c_int32),
                ("chunks", ctypes.c_int32), ("split_k", ctypes.c_int32),
                ("k_split", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("device", ctypes.c_int32),
                ("conv_rows_per_tile", ctypes.c_int32), ("conv_images_per_tile", ctypes.c_int32),
                ("max_panel_nnz", ctypes.c_int64), ("min_panel_nnz", ctypes.c_int64),
                ("build_ms", ctypes.c_double), ("executor", ctypes.c_int32),
                ("jit_modules", ctypes.c_int32), ("jit_rows", ctypes.c_int32),
                ("jit_warps", ctypes.c_int32), ("jit_cubin_bytes", ctypes.c_int64),
                ("jit_compile_ms", ctypes.c_double), ("tuned_us", ctypes.c_double),
                ("digest", ctypes.c_uint64), ("x_multicast", ctypes.c_int32),
                ("x_source", ctypes.c_int32), ("conv_kernel", ctypes.c_int32),
                ("row_order", ctypes.c_int32), ("tc_min_density", ctypes.c_int32),
                ("tc_row_blocks", ctypes.c_int32), ("tc_tiles", ctypes.c_int64),
                ("tc_nnz", ctypes.c_int64), ("tc_panel_steps", ctypes.c_int64),
                ("plan_source", ctypes.c_int32), ("cta_pair", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.sparse_plan_opts_init.argtypes = [ctypes.POINTER(sparse_plan_opts)]
    lib.sparse_plan_opts_init.restype = None
    lib.sparse_plan_create.argtypes = [ctypes.POINTER(P), i32, i32, i64, P, P, P, i32,
                                       ctypes.POINTER(sparse_plan_opts)]
    lib.sparse_plan_create.restype = ctypes.c_int
    lib.sparse_spmm.argtypes = [P, i64, P, i64, P, i64, P]
    lib.sparse_spmm.restype = ctypes.c_int
    lib.sparse_conv3x3.argtypes = [P, i64, P, P, P]
    lib.sparse_linear.argtypes = [P, i64, P, i64, P, i64, P]
    lib.sparse_conv3x3.restype = ctypes.c_int
    lib.sparse_spmm_ex.argtypes = [P, i64, P, i64, P, i64, ctypes.POINTER(sparse_epilogue), P]
    lib.sparse_spmm_ex.restype = ctypes.c_int
    lib.sparse_conv3x3_ex.argtypes = [P, i64, P, P, ctypes.POINTER(sparse_epilogue), P]
    lib.sparse_conv3x3_ex.restype = ctypes.c_int
    lib.sparse_conv1x1.argtypes = [P, i64, i32, i32, i32, P, P, P]
    lib.sparse_conv1x1.restype = ctypes.c_int
    lib.sparse_conv3x3_nhwc.argtypes = [P, i64, P, P, P]
    lib.sparse_conv3x3_nhwc.restype = ctypes.c_int
    lib.plan_destroy.argtypes = [P]
    lib.plan_destroy.restype = ctypes.c_int
    lib.sparse_plan_destroy.argtypes = [P]
    lib.sparse_plan_destroy.restype = ctypes.c_int
    lib.sparse_plan_info.argtypes = [P, ctypes.POINTER(sparse_plan_info_t)]
    lib.sparse_plan_info.restype = ctypes.c_int
    lib.sparse_plan_dump.argtypes = [P, i64, P, P, P, P, P, P, P]
    lib.sparse_plan_dump.restype = ctypes.c_int
    lib.sparse_last_error.argtypes = []
    lib.sparse_last_error.restype = ctypes.c_char_p
    lib.sparse_version.argtypes = []
    lib.sparse_version.restype = ctypes.c_char_p
    return lib


lib = _load()


def _check(rc: int):
    if rc != SPARSE_OK:
        raise SparseRTError(rc, lib.sparse_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- C names

def sparse_plan_create(M, K, row_ptr, col_idx, values, dtype=SPARSE_F32, **opts) -> ctypes.c_void_p:
    """Run the inspector and upload the plan; returns the opaque handle."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.float32)
    o = sparse_plan_opts()
    lib.sparse_plan_opts_init(ctypes.byref(o))
    for k, val in opts.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown plan option {k}")
        setattr(o, k, int(val))
    h = ctypes.c_void_p()
    nnz = int(rp[-1]) if rp.size else 0
    _check(lib.sparse_plan_create(ctypes.byref(h), int(M), int(K), nnz, _ptr(rp),
                                  _ptr(ci) if ci.size else None, _ptr(v) if v.size else None,
                                  int(dtype), ctypes.byref(o)))
    return h


def sparse_spmm(plan, N, X_ptr, ldx, Y_ptr, ldy, stream=0):
    _check(lib.sparse_spmm(plan, int(N), X_ptr, int(ldx), Y_ptr, int(ldy), stream))


def sparse_linear(plan, N, X_ptr, ldx, Y_ptr, ldy, stream=0):
    _check(lib.sparse_linear(plan, int(N), X_ptr, int(ldx), Y_ptr, int(ldy), stream))


def sparse_conv3x3(plan, batch, x_ptr, y_ptr, stream=0):
    _check(lib.sparse_conv3x3(plan, int(batch), x_ptr, y_ptr, stream))


def sparse_spmm_ex(plan, N, X_ptr, ldx, Y_ptr, ldy, epilogue=None, stream=0):
    ep = ctypes.byref(epilogue) if epilogue is not None else None
    _check(lib.sparse_spmm_ex(plan, int(N), X_ptr, int(ldx), Y_ptr, int(ldy), ep, stream))


def sparse_conv3x3_ex(plan, batch, x_ptr, y_ptr, epilogue=None, stream=0):
    ep = ctypes.byref(epilogue) if epilogue is not None else None
    _check(lib.sparse_conv3x3_ex(plan, int(batch), x_ptr, y_ptr, ep, stream))


def sparse_conv1x1(plan, batch, h, w, stride, x_ptr, y_ptr, stream=0):
    _check(lib.sparse_conv1x1(plan, int(batch), int(h), int(w), int(stride), x_ptr, y_ptr, stream))


def sparse_conv3x3_nhwc(plan, batch, x_ptr, y_ptr, stream=0):
    _check(lib.sparse_conv3x3_nhwc(plan, int(batch), x_ptr, y_ptr, stream))


def plan_destroy(plan):
    _check(lib.plan_destroy(plan))


def sparse_plan_info(plan) -> dict:
    info = sparse_plan_info_t()
    _check(lib.sparse_plan_info(plan, ctypes.byref(info)))
    return {name: getattr(info, name) for name, _ in info._fields_}


@dataclass
class PlanDump:
    row: np.ndarray
    col: np.ndarray
    value: np.ndarray
    panel: np.ndarray
    chunk: np.ndarray
    slot: np.ndarray
    group: np.ndarray


def sparse_plan_dump(plan) -> PlanDump:
    nnz = sparse_plan_info(plan)["nnz"]
    arrs = [np.zeros(max(nnz, 1), np.int32) for _ in range(2)]
    val = np.zeros(max(nnz, 1), np.float32)
    more = [np.zeros(max(nnz, 1), np.int32) for _ in range(4)]
    _check(lib.sparse_plan_dump(plan, max(nnz, 1), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(val),
                                *[_ptr(a) for a in more]))
    return PlanDump(arrs[0][:nnz], arrs[1][:nnz], val[:nnz], *[a[:nnz] for a in more])


def version() -> str:
    return lib.sparse_version().decode()


# ----------------------------------------------------------------------------- torch API

_TORCH_DT = {}


def _dtype_code(t) -> int:
    import torch
    if t == torch.float32:
        return SPARSE_F32
    if t == torch.float16:
        return SPARSE_F16
    if t == torch.bfloat16:
        return SPARSE_BF16
    raise TypeError(f"unsupported dtype {t}")


class Plan:
    """Owning wrapper: Plan(csr_or_arrays, dtype=torch.float32, **opts).

    `opts` are sparse_plan_opts fields (kind, c_in, h, w, n_hint, device, drop_zeros,
    warps, rows_per_warp, k_chunk, split_k).  Use device=SPARSE_DEVICE_HOST_ONLY for an
    inspect-only plan on a machine without a GPU.
    """

    def __init__(self, M, K, row_ptr, col_idx, values, dtype=None, **opts):
        import torch
        dtype = torch.float32 if dtype is None else dtype
        self.dtype = dtype
        self.M, self.K = int(M), int(K)
        self.kind = int(opts.get("kind", SPARSE_SPMM))
        self.conv_geom = (opts.get("c_in", 0), opts.get("h", 0), opts.get("w", 0))
        self._h = sparse_plan_create(M, K, row_ptr, col_idx, values, _dtype_code(dtype), **opts)
        self.info = sparse_plan_info(self._h)

    @classmethod
    def from_csr(cls, csr, dtype=None, **opts):
        return cls(csr.M, csr.K, csr.row_ptr, csr.col_idx, csr.values, dtype=dtype, **opts)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h is not None and self._h.value:
            plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dump(self) -> PlanDump:
        return sparse_plan_dump(self._h)

    def chosen_opts(self) -> dict:
        """The tile options this plan was built with (e.g. after tune=1): passing them to
        another Plan of the same matrix rebuilds an identical replica (same digest)."""
        i = self.info
        o = dict(warps=i["warps"], rows_per_warp=i["rows_per_warp"], split_k=i["split_k"],
                 stages=i["stages"], executor=i["executor"], row_order=i["row_order"])
        if self.kind == SPARSE_SPMM:
            o.update(k_chunk=i["k_chunk"], k_split=i["k_split"], x_multicast=i["x_multicast"],
                     x_source=i["x_source"], tc_min_density=i["tc_min_density"] or -1)
            if i["executor"] == 1:
                o.update(jit_rows=i["jit_rows"], jit_warps=i["jit_warps"])
            if i["plan_source"]:
                o.update(plan_source=i["plan_source"])
            if i["executor"] == 4:  # the tcgen05 block executor has its own fixed ring
                o.pop("stages")
                if i["cta_pair"]:
                    o.update(cta_pair=1)
        else:
            o.update(k_chunk=i["k_chunk"], conv_kernel=i["conv_kernel"])
            o.pop("split_k")
            o.pop("stages")
            if i["conv_kernel"] == 5:  # tcgen05 blocks: the tile options are the executor's own
                o = dict(conv_kernel=5, x_multicast=i["x_multicast"])
                if i["cta_pair"]:
                    o.update(cta_pair=1)
        return o

    def _check_tensor(self, t, name):
        import torch
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype != self.dtype:
            raise TypeError(f"{name} dtype {t.dtype} != plan dtype {self.dtype}")
        dev = self.info["device"]
        if t.device.index != dev:
            raise ValueError(f"{name} on {t.device}, plan on cuda:{dev}")

    def _epilogue(self, bias, beta, relu, n_out):
        if bias is None and beta == 0.0 and not relu:
            return None
        if bias is not None:
            self._check_tensor(bias, "bias")
            if bias.dim() != 1 or bias.shape[0] != n_out or not bias.is_contiguous():
                raise ValueError(f"bias must be a contiguous vector of {n_out} values")
        return sparse_epilogue(float(beta), ctypes.c_void_p(bias.data_ptr()) if bias is not None else None,
                               1 if relu else 0)

    def spmm(self, X, Y=None, stream=None, bias=None, beta=0.0, relu=False):
        """Y[:, :N] = act(W @ X + bias + beta * Y).  X: (K, N) CUDA tensor with unit column
        stride (row stride = ldx); bias: (M,) plan dtype; relu: ReLU after the sum."""
        import torch
        if self.kind != SPARSE_SPMM:
            raise ValueError("spmm on a conv plan")
        self._check_tensor(X, "X")
        if X.dim() != 2 or X.shape[0] != self.K or (X.shape[1] > 1 and X.stride(1) != 1):
            raise ValueError("X must be (K, N) with unit column stride")
        N = X.shape[1]
        if beta != 0.0 and Y is None:
            raise ValueError("beta != 0 needs Y")
        if Y is None:
            Y = torch.empty((self.M, N), dtype=self.dtype, device=X.device)
        self._check_tensor(Y, "Y")
        if Y.dim() != 2 or Y.shape[0] != self.M or Y.shape[1] != N or (N > 1 and Y.stride(1) != 1):
            raise ValueError("Y must be (M, N) with unit column stride")
        s = (stream or torch.cuda.current_stream(X.device)).cuda_stream
        ldx = X.stride(0) if N > 0 else max(N, 1)
        ldy = Y.stride(0) if N > 0 else max(N, 1)
        ep = self._epilogue(bias, beta, relu, self.M)
        if ep is None:
            sparse_spmm(self._h, N, ctypes.c_void_p(X.data_ptr()), max(ldx, N),
                        ctypes.c_void_p(Y.data_ptr()), max(ldy, N), ctypes.c_void_p(s))
        else:
            sparse_spmm_ex(self._h, N, ctypes.c_void_p(X.data_ptr()), max(ldx, N),
                           ctypes.c_void_p(Y.data_ptr()), max(ldy, N), ep, ctypes.c_void_p(s))
        return Y

    def linear(self, X, Y=None, stream=None):
        """Token-major layout (nn.Linear): Y (N, M) = X (N, K) @ W^T, rows contiguous."""
        import torch
        if self.kind != SPARSE_SPMM:
            raise ValueError("linear on a conv plan")
        self._check_tensor(X, "X")
        if X.dim() != 2 or X.shape[1] != self.K or (self.K > 1 and X.stride(1) != 1):
            raise ValueError("X must be (N, K) with unit column stride")
        N = X.shape[0]
        if Y is None:
            Y = torch.empty((N, self.M), dtype=self.dtype, device=X.device)
        self._check_tensor(Y, "Y")
        if Y.dim() != 2 or Y.shape != (N, self.M) or (self.M > 1 and Y.stride(1) != 1):
            raise ValueError("Y must be (N, M) with unit column stride")
        s = (stream or torch.cuda.current_stream(X.device)).cuda_stream
        sparse_linear(self._h, N, ctypes.c_void_p(X.data_ptr()), max(X.stride(0), self.K),
                      ctypes.c_void_p(Y.data_ptr()), max(Y.stride(0), self.M), ctypes.c_void_p(s))
        return Y

    def conv3x3(self, x, y=None, stream=None, bias=None, beta=0.0, relu=False):
        """y = act(conv3x3(x) + bias + beta * y), x: (C_in, B, H, W) contiguous CUDA tensor
        (CNHW); bias: (C_out,) plan dtype."""
        import torch
        if self.kind != SPARSE_CONV3X3:
            raise ValueError("conv3x3 on an SpMM plan")
        self._check_tensor(x, "x")
        c_in, h, w = self.conv_geom
        if x.dim() != 4 or tuple(x.shape[0:1]) + tuple(x.shape[2:]) != (c_in, h, w) or not x.is_contiguous():
            raise ValueError(f"x must be contiguous (C_in={c_in}, B, H={h}, W={w})")
        B = x.shape[1]
        if beta != 0.0 and y is None:
            raise ValueError("beta != 0 needs y")
        if y is None:
            y = torch.empty((self.M, B, h, w), dtype=self.dtype, device=x.device)
        self._check_tensor(y, "y")
        if tuple(y.shape) != (self.M, B, h, w) or not y.is_contiguous():
            raise ValueError("y must be contiguous (C_out, B, H, W)")
        s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
        ep = self._epilogue(bias, beta, relu, self.M)
        if ep is None:
            sparse_conv3x3(self._h, B, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                           ctypes.c_void_p(s))
        else:
            sparse_conv3x3_ex(self._h, B, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                              ep, ctypes.c_void_p(s))
        return y

    def conv1x1(self, x, stride=1, y=None, stream=None):
        """Strided 1x1 convolution on an SpMM plan of W (C_out x C_in): x (C_in, B, h, w) CNHW ->
        y (C_out, B, ceil(h/stride), ceil(w/stride)), y[co, b, oy, ox] = sum W[co, ci] x[ci, b, oy s, ox s]."""
        import torch
        if self.kind != SPARSE_SPMM:
            raise ValueError("conv1x1 needs an SpMM plan")
        self._check_tensor(x, "x")
        if x.dim() != 4 or x.shape[0] != self.K or not x.is_contiguous():
            raise ValueError(f"x must be contiguous (C_in={self.K}, B, h, w)")
        _, B, h, w = x.shape
        ho, wo = (h + stride - 1) // stride, (w + stride - 1) // stride
        if y is None:
            y = torch.empty((self.M, B, ho, wo), dtype=self.dtype, device=x.device)
        self._check_tensor(y, "y")
        if tuple(y.shape) != (self.M, B, ho, wo) or not y.is_contiguous():
            raise ValueError("y must be contiguous (C_out, B, ho, wo)")
        s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
        sparse_conv1x1(self._h, B, h, w, stride, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                       ctypes.c_void_p(s))
        return y

    def conv3x3_nhwc(self, x, y=None, stream=None):
        """Channels-last 3x3 conv: x (B, H, W, C_in) -> y (B, H, W, C_out), contiguous."""
        import torch
        if self.kind != SPARSE_CONV3X3:
            raise ValueError("conv3x3_nhwc on an SpMM plan")
        self._check_tensor(x, "x")
        c_in, h, w = self.conv_geom
        if x.dim() != 4 or tuple(x.shape[1:]) != (h, w, c_in) or not x.is_contiguous():
            raise ValueError(f"x must be contiguous (B, H={h}, W={w}, C_in={c_in})")
        B = x.shape[0]
        if y is None:
            y = torch.empty((B, h, w, self.M), dtype=self.dtype, device=x.device)
        self._check_tensor(y, "y")
        if tuple(y.shape) != (B, h, w, self.M) or not y.is_contiguous():
            raise ValueError("y must be contiguous (B, H, W, C_out)")
        s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
        sparse_conv3x3_nhwc(self._h, B, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                            ctypes.c_void_p(s))
        return y
