"""paper_2008_11849_b200 — B200-native SparseRT hot path (arXiv 2008.11849).

Y = W @ X for a pruned, unstructured-sparse W (CSR in) and dense X, plus sparse 3x3
convolution through implicit im2col, executed by hand-written sm_100a CUDA kernels in
libsparsert.so behind the C ABI of include/sparsert.h.  This package is the thin Python
binding (ctypes); see DESIGN.md.
"""
from .sparsert import (  # noqa: F401
    SPARSE_CONV3X3, SPARSE_DEVICE_HOST_ONLY, SPARSE_F16, SPARSE_F32, SPARSE_SPMM, Plan,
    SparseRTError, lib, plan_destroy, sparse_conv3x3, sparse_plan_create, sparse_plan_dump,
    sparse_plan_info, sparse_spmm, version, sparse_spmm_ex, sparse_conv3x3_ex, sparse_epilogue,
    sparse_linear,
)
