"""Multi-GPU plumbing: one process per GPU, images sharded, no collective on
the data path.

The SpMM of each image depends only on that image's [K][H*W] block, so a
batch splits into contiguous image ranges, one per rank, with the weights
replicated (they are at most ~1 MB). torch.distributed is used only for the
timing barrier and the max-over-ranks of the measured time.
"""
from __future__ import annotations

import os


def shard(images: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) image range of `rank` out of `world`; sizes
    differ by at most one and the ranges tile [0, images) exactly."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(images, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


class Dist:
    """RANK/WORLD_SIZE/LOCAL_RANK from the environment (torchrun); a process
    group only when WORLD_SIZE > 1."""

    def __init__(self, backend: str = "nccl"):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if not dist.is_initialized():
                dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self, device=None):
        if self.pg:
            if device is not None and self.backend == "nccl":
                self.pg.barrier(device_ids=[device])
            else:
                self.pg.barrier()

    def max(self, x: float, device=None) -> float:
        """Max of a scalar over ranks (timing only)."""
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64,
                         device=device if (device is not None and self.backend == "nccl") else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float, device=None) -> float:
        """Sum of a scalar over ranks (work accounting only)."""
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64,
                         device=device if (device is not None and self.backend == "nccl") else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg and self.pg.is_initialized():
            self.pg.destroy_process_group()
