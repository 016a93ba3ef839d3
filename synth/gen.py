"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no SpMM, no convolution, no plan logic).
It only draws inputs: magnitude-pruned weight matrices in CSR form and dense activations,
with the shapes / sparsities of the paper's workloads (Table 1 P:224-254,
Table 3, BASELINE.json configs).  Recipe:

* W: dense w ~ N(0, 2/K) (He-normal), keep exactly nnz = round_half_up((100-p)*M*K/100)
  largest |w| (ties -> lower flat index), the rest are structural zeros.  The paper used
  "pruned weights from real neural networks", observed to be "quite uniform"
  (P:385); magnitude pruning of an i.i.d. matrix gives uniform positions.
* X (SpMM): U(-1, 1).  X (conv): ReLU(N(0,1)) (post-activation data).
* Exact mode: small integers so every fp32 partial sum is exact (< 2^24).
* Stress patterns (parity only): skewed rows, empty rows, dense row, block-dense, one column.

numpy PCG64 (`np.random.default_rng(seed)`) everywhere; seeds are explicit arguments.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Csr:
    """CSR matrix (M x K): row_ptr int32[M+1], col_idx int32[nnz], values float32[nnz]."""
    M: int
    K: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def with_values(self, values: np.ndarray) -> "Csr":
        return Csr(self.M, self.K, self.row_ptr, self.col_idx,
                   np.ascontiguousarray(values, dtype=np.float32))


def nnz_for(M: int, K: int, sparsity_pct: float) -> int:
    """nnz = round_half_up((100 - p) * M * K / 100) in exact integer arithmetic when p is
    integral (SURVEY 8(c) reading #10: "% nnz" column of Table 1 holds the sparsity)."""
    if float(sparsity_pct).is_integer():
        p = int(sparsity_pct)
        return ((100 - p) * M * K * 2 + 100) // 200
    return int(np.floor((100.0 - sparsity_pct) * M * K / 100.0 + 0.5))


def csr_from_mask(M: int, K: int, flat_keep: np.ndarray, values_dense: np.ndarray) -> Csr:
    """Build CSR from the sorted flat indices to keep (row-major m*K+k)."""
    flat_keep = np.sort(np.asarray(flat_keep, dtype=np.int64))
    rows = flat_keep // K
    cols = flat_keep % K
    row_ptr = np.zeros(M + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    vals = values_dense.reshape(-1)[flat_keep].astype(np.float32)
    return Csr(M, K, row_ptr, cols.astype(np.int32), vals)


def pruned_weights(M: int, K: int, sparsity_pct: float, seed: int) -> Csr:
    """Magnitude-pruned He-normal W (M x K) with exactly nnz_for(M, K, p) nonzeros."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((M, K)) * np.sqrt(2.0 / K)
    nnz = nnz_for(M, K, sparsity_pct)
    order = np.argsort(-np.abs(w).reshape(-1), kind="stable")  # ties: lower flat index first
    keep = order[:nnz]
    csr = csr_from_mask(M, K, keep, w.astype(np.float32))
    # a magnitude-pruned value is never exactly zero in float32 unless underflow; guard anyway
    z = csr.values == 0
    if z.any():
        csr.values[z] = np.float32(1e-3)
    return csr


def uniform_x(K: int, N: int, seed: int, ld: int | None = None) -> np.ndarray:
    """X ~ U(-1, 1), float32, shape (K, ld) with the first N columns meaningful (ld >= N)."""
    rng = np.random.default_rng(seed)
    ld = N if ld is None else ld
    x = rng.uniform(-1.0, 1.0, size=(K, ld)).astype(np.float32)
    return x


def relu_normal_x(shape, seed: int) -> np.ndarray:
    """Conv input: ReLU(N(0,1)) float32 of the given shape (CNHW)."""
    rng = np.random.default_rng(seed)
    return np.maximum(rng.standard_normal(shape), 0.0).astype(np.float32)


def int_weights(M: int, K: int, sparsity_pct: float, seed: int, vmax: int = 3) -> Csr:
    """Exact-mode W: same positions as pruned_weights, values in {+-1..+-vmax}."""
    csr = pruned_weights(M, K, sparsity_pct, seed)
    rng = np.random.default_rng(seed + 7919)
    mag = rng.integers(1, vmax + 1, size=csr.nnz)
    sgn = rng.choice(np.array([-1, 1]), size=csr.nnz)
    return csr.with_values((mag * sgn).astype(np.float32))


def int_x(K: int, N: int, seed: int, vmax: int = 3, ld: int | None = None) -> np.ndarray:
    """Exact-mode X: integers in [-vmax, vmax], float32, shape (K, ld)."""
    rng = np.random.default_rng(seed)
    ld = N if ld is None else ld
    return rng.integers(-vmax, vmax + 1, size=(K, ld)).astype(np.float32)


def random_pattern(M: int, K: int, nnz: int, seed: int, values: str = "normal") -> Csr:
    """Uniformly random positions (without replacement), given nnz."""
    rng = np.random.default_rng(seed)
    keep = rng.choice(M * K, size=nnz, replace=False) if nnz > 0 else np.zeros(0, np.int64)
    if values == "normal":
        v = rng.standard_normal(M * K).astype(np.float32)
        v[v == 0] = 1.0
    else:
        v = rng.integers(1, 4, size=M * K).astype(np.float32) * rng.choice([-1.0, 1.0], size=M * K).astype(np.float32)
    return csr_from_mask(M, K, keep, v)


def stress_pattern(kind: str, M: int, K: int, seed: int, density: float = 0.1) -> Csr:
    """Stress patterns for parity: 'zipf', 'empty_rows', 'dense_row',
    'block_dense', 'block16', 'one_column', 'empty'.  'block16': a fraction `density` of the
    aligned 16x16 tiles fully dense plus uniform 5% background nonzeros (the structured case
    of the tensor-core sub-block path)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((M, K)).astype(np.float32)
    v[v == 0] = 1.0
    if kind == "empty":
        return Csr(M, K, np.zeros(M + 1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32))
    if kind == "zipf":
        total = max(1, int(round(density * M * K)))
        wts = 1.0 / np.arange(1, M + 1) ** 1.2
        wts = wts[rng.permutation(M)]
        per = np.minimum(K, np.floor(wts / wts.sum() * total).astype(np.int64))
        keep = []
        for m in range(M):
            cols = rng.choice(K, size=int(per[m]), replace=False)
            keep.append(m * K + cols)
        keep = np.concatenate(keep) if keep else np.zeros(0, np.int64)
        return csr_from_mask(M, K, keep, v)
    if kind == "empty_rows":
        mask = rng.random((M, K)) < density
        mask[rng.random(M) < 0.1, :] = False
        return csr_from_mask(M, K, np.flatnonzero(mask), v)
    if kind == "dense_row":
        mask = rng.random((M, K)) < density
        mask[rng.integers(0, M), :] = True
        return csr_from_mask(M, K, np.flatnonzero(mask), v)
    if kind == "block_dense":
        mask = np.zeros((M, K), bool)
        nb = max(1, int(density * (M // 8) * (K // 8)))
        bi = rng.choice((M // 8) * (K // 8), size=nb, replace=False)
        for b in bi:
            r, c = divmod(int(b), K // 8)
            mask[r * 8:(r + 1) * 8, c * 8:(c + 1) * 8] = True
        return csr_from_mask(M, K, np.flatnonzero(mask), v)
    if kind == "block16":
        mask = rng.random((M, K)) < 0.05
        nrb, ncb = M // 16, K // 16
        nb = max(1, int(density * nrb * ncb))
        for b in rng.choice(nrb * ncb, size=nb, replace=False):
            r, c = divmod(int(b), ncb)
            mask[r * 16:(r + 1) * 16, c * 16:(c + 1) * 16] = True
        return csr_from_mask(M, K, np.flatnonzero(mask), v)
    if kind == "one_column":
        mask = np.zeros((M, K), bool)
        mask[:, rng.integers(0, K)] = True
        return csr_from_mask(M, K, np.flatnonzero(mask), v)
    raise ValueError(kind)


def identity_csr(n: int) -> Csr:
    return Csr(n, n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
               np.ones(n, np.float32))


def row_selection_csr(M: int, K: int, seed: int) -> Csr:
    """Each row m has a single 1 at column sigma(m) (sigma arbitrary)."""
    rng = np.random.default_rng(seed)
    sigma = rng.integers(0, K, size=M).astype(np.int32)
    return Csr(M, K, np.arange(M + 1, dtype=np.int32), sigma, np.ones(M, np.float32))


def to_dense(csr: Csr, dtype=np.float64) -> np.ndarray:
    """Scatter CSR into a dense array (input plumbing for tests; not the oracle's SpMM)."""
    d = np.zeros((csr.M, csr.K), dtype=dtype)
    rows = np.repeat(np.arange(csr.M), np.diff(csr.row_ptr))
    d[rows, csr.col_idx] = csr.values
    return d


# --------------------------------------------------------------------------------------
# Workload catalogue (BASELINE.json configs; Table 1 / Table 3)
# --------------------------------------------------------------------------------------

# Table 1: problem id -> (M, K, N at batch 1)
TABLE1 = {
    1: (64, 256, 3136), 2: (256, 64, 3136), 3: (128, 512, 784), 4: (512, 128, 784),
    5: (256, 1024, 196), 6: (1024, 256, 196), 7: (512, 2048, 49), 8: (2048, 512, 49),
    9: (2048, 512, 256), 10: (512, 2048, 256), 11: (512, 512, 256),
    12: (64, 32, 12544), 13: (128, 64, 3136), 14: (128, 128, 3136), 15: (256, 128, 784),
    16: (256, 256, 784), 17: (512, 256, 196), 18: (512, 512, 196), 19: (1024, 512, 49),
    20: (1024, 1024, 49),
}
RN50_1X1 = [1, 2, 3, 4, 5, 6, 7, 8]
MBV1_PW = [12, 13, 14, 15, 16, 17, 18, 19, 20]
BERT_FC = [(3072, 768), (768, 3072)]
# Table 3: (H=W, C_in=C_out)
TABLE3 = {1: (56, 64), 2: (28, 128), 3: (14, 256), 4: (7, 512)}


def case_seed(name: str, salt: int = 0) -> int:
    """Stable per-case seed derived from the case name (no hash randomisation)."""
    h = 2166136261
    for ch in name.encode():
        h = ((h ^ ch) * 16777619) & 0xFFFFFFFF
    return (h + salt) & 0x7FFFFFFF
