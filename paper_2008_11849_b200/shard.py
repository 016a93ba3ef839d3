"""N-sharding for multi-GPU runs: Y[:, n] = W X[:, n], so columns are
independent and each rank takes a contiguous column slab with a replicated plan; no collective
is needed on the data path.  Slab boundaries fall on whole samples (`unit` columns: H*W for
images, seq for sequences) so a 3x3 convolution never needs a halo exchange."""
from __future__ import annotations


def shard_columns(n_total: int, world: int, rank: int, unit: int = 1) -> tuple[int, int]:
    """Half-open column range [n0, n1) of `rank`: whole units, as even as possible, the first
    (n_units % world) ranks taking one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if unit < 1 or n_total % unit:
        raise ValueError("n_total must be a multiple of unit")
    units = n_total // unit
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return u0 * unit, u1 * unit


def gather_columns(y_local, n_total: int, world: int, unit: int = 1, group=None):
    """Optional gather of the N-sharded outputs: every rank receives the full
    (rows, n_total) tensor assembled from the ranks' column slabs (shard_columns layout).
    One all_gather over slabs padded to the largest slab (NCCL over NVLink / NVSwitch on GPU,
    gloo on CPU), then the padding is dropped.  Off the data path: the SpMM itself needs no
    exchange, so callers time this separately."""
    import torch
    import torch.distributed as dist
    rows = y_local.shape[0]
    sizes = [shard_columns(n_total, world, r, unit) for r in range(world)]
    width = max(b - a for a, b in sizes)
    buf = torch.zeros((rows, width), dtype=y_local.dtype, device=y_local.device)
    buf[:, :y_local.shape[1]] = y_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    return torch.cat([p[:, :b - a] for p, (a, b) in zip(parts, sizes)], dim=1)
