"""Data parallelism over one node: one process per GPU, NCCL over NVLink.

Mini-batches shard naturally: a batch's samples
depend only on ``derive_seed(seed, 13, j)`` (trainer.py:304), so rank r takes
windows ``w = r, r + W, ...`` and keeps its own Match-Reorder state.  The only
exchange is one flat fp32 gradient bucket per step (all weights and biases,
DeviceModel.grad), averaged with one all-reduce before SGD -- synchronous DP
on the mean of W batch gradients.
"""

from __future__ import annotations

import os


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init(backend: str = "nccl"):
    """Initialise torch.distributed from torchrun's environment (127.0.0.1 rendezvous)."""
    import torch.distributed as dist
    rank, world, _ = env_rank()
    if world > 1 and not dist.is_initialized():
        # the gradient all-reduce is captured into CUDA graphs: the NCCL
        # watchdog must not query events of captured work
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "0")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world


def shard(items, rank: int, world: int):
    """Round-robin shard of windows: rank r gets items r, r+W, r+2W, ..."""
    return items[rank::world]


def lockstep_count(n_local: int, world: int, device=None) -> int:
    """Number of steps every rank can take together (min over ranks)."""
    if world <= 1:
        return n_local
    import torch
    import torch.distributed as dist
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item())


class GradAllReduce:
    """Sums the flat gradient bucket across ranks (one collective per step);
    the trainer folds the 1/W of the mean into the SGD step (lr / W).

    With the NCCL backend the collective is issued on the caller's current
    stream and can be captured into the trainer's CUDA graphs (NCCL >= 2.9.6
    supports stream capture; the communicator is created by ``warmup``
    before any capture, and the watchdog's asynchronous error handling must
    be off: TORCH_NCCL_ASYNC_ERROR_HANDLING=0, set by ``init``).  gloo
    (CPU tests, several ranks sharing one GPU) cannot be captured; the
    trainer then runs eagerly."""

    def __init__(self, world: int):
        self.world = int(world)
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist
            self.backend = str(dist.get_backend())
        self.capturable = self.backend == "nccl"
        self._warm = False

    def warmup(self, device=None):
        """One eager collective: creates the communicator outside any capture."""
        if self.world <= 1 or self._warm:
            return
        import torch
        import torch.distributed as dist
        t = torch.zeros(1, dtype=torch.float32, device=device)
        dist.all_reduce(t)
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        self._warm = True

    def allreduce_sum(self, flat):
        if self.world <= 1:
            return
        import torch.distributed as dist
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)

    def allreduce_mean(self, flat):
        if self.world <= 1:
            return
        self.allreduce_sum(flat)
        flat.mul_(1.0 / self.world)


def max_over_ranks(value: float, world: int, device=None) -> float:
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, world: int, device=None) -> float:
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
