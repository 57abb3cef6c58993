"""Z-slab sharding of the SLIC iteration loop across GPUs (one process per GPU).

Decomposition: the last (slowest) axis is split into contiguous
slabs, one per rank. Assignment needs no image halo because every rank holds
the full (small) centre table; only the one-time perturbation reads a 2-plane
halo. The single data-path exchange per iteration is an allreduce of the
per-cluster int64 partial sums — integer addition is associative, so results
are bitwise identical for 1/2/4/8 ranks (the analogue of the reference's
"bitwise identical for any worker count", parallel.hpp:1-8).

The driver is written against two small protocols so the same code runs the
CUDA engine over NCCL on B200s and an oracle-backed engine over gloo on CPU
(tests/test_sharded_gloo.py):

* engine: init(), centers_tensor(), commit(), assign(), partials_tensor(),
  update();
* allreduce(tensor): in-place SUM across ranks (torch.distributed).
"""
from __future__ import annotations

from typing import Optional, Callable, List, Tuple


def slab_bounds(last: int, world: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous near-equal split of [0, last) into `world` slabs; slab
    boundaries are rounded to multiples of `align` planes when possible."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = (last + align - 1) // align
    if units < world:
        align, units = 1, last
    lo = (units * rank) // world * align
    hi = (units * (rank + 1)) // world * align
    return min(lo, last), min(hi, last)


def data_bounds(last: int, slab: Tuple[int, int], halo: int = 2) -> Tuple[int, int]:
    """Planes a rank must hold: its slab plus the perturbation halo."""
    return max(0, slab[0] - halo), min(last, slab[1] + halo)


def all_slabs(last: int, world: int, align: int = 1) -> List[Tuple[int, int]]:
    return [slab_bounds(last, world, r, align) for r in range(world)]


def _dist_max(v: float) -> float:
    """MAX of a scalar over the torch.distributed group (NCCL: on the
    current CUDA device; gloo: on the CPU)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ShardedLoop:
    """run_slic's loop (slic.hpp:397-412) over one slab per rank."""

    def __init__(self, engine, allreduce: Callable, world: int,
                 allreduce_max: Optional[Callable[[float], float]] = None):
        self.engine = engine
        self.allreduce = allreduce
        self.world = world
        self.allreduce_max = allreduce_max or _dist_max

    def init(self):
        """init + perturb: every rank fills the clusters whose initial cell
        centre lies in its slab and zeros elsewhere; the SUM allreduce then
        assembles the full table exactly (one non-zero term per entry).
        First, every rank adopts the MAX over ranks of the engines' value
        ranges: the fixed-point scale of the allreduced float sums must be
        one scale (sslic_engine_set_value_range)."""
        if self.world > 1 and hasattr(self.engine, "value_range"):
            self.engine.set_value_range(self.allreduce_max(self.engine.value_range()))
        self.engine.init()
        if self.world > 1:
            self.allreduce(self.engine.centers_tensor())
        self.engine.commit()

    def gather_labels(self, gather: Callable, last: int, plane: int, align: int = 1,
                      rank: int = 0, dst: int = 0):
        """The full label map on rank `dst` only (None elsewhere): each rank
        sends its slab (engine.labels_tensor(), padded to the largest slab so
        the collective sees equal sizes) and `dst` concatenates them along the
        last axis in rank order. `gather(tensor, parts_or_None, dst)` is
        torch.distributed.gather(tensor, gather_list, dst)."""
        import torch
        slabs = all_slabs(last, self.world, align)
        mine = self.engine.labels_tensor()
        width = max(hi - lo for lo, hi in slabs) * plane
        buf = torch.zeros(width, dtype=mine.dtype, device=mine.device)
        buf[: mine.numel()] = mine
        parts = [torch.empty_like(buf) for _ in range(self.world)] if rank == dst else None
        gather(buf, parts, dst)
        if rank != dst:
            return None
        return torch.cat([parts[r][: (hi - lo) * plane] for r, (lo, hi) in enumerate(slabs)])

    def segment(self, gather: Callable, connectivity: Callable, last: int, plane: int,
                align: int = 1, rank: int = 0, dst: int = 0):
        """enforce_connectivity over the sharded result on rank `dst`: the
        slabs are gathered there (one copy of the map, not one per rank) and
        `connectivity(full)` runs once -- on a B200 the device pass handles
        2^32+ voxels with its own slab stitching (connectivity.cu), so a
        config-5 map fits one GPU. Other ranks return None."""
        full = self.gather_labels(gather, last, plane, align, rank, dst)
        return None if full is None else connectivity(full)

    def iterate(self):
        """One iteration: fused assign+accumulate on the slab, SUM of the
        int64 partials, identical update on every rank."""
        self.engine.assign()
        if self.world > 1:
            self.allreduce(self.engine.partials_tensor())
        self.engine.update()
