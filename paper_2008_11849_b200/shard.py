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
