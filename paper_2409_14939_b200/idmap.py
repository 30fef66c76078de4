"""Fused-Map ID table: drop-in for ``minigl.idmap`` backed by csrc/idmap.cu.

``build`` returns an :class:`IdMapTable` whose keys/values (host uint64
arrays, like the reference) hold exactly the single-worker reference state:
first-seen local IDs and the sequential linear-probing slot layout for both
hash kinds (idmap.py:88-117, :175-233).  ``workers`` is accepted for API
compatibility; the GPU build is parallel and deterministic for any value.

On the trainer path this table is not needed at all: the window sampler
assigns local IDs as ranks in the sorted unique set while it samples
(csrc/sampler.cu), which is what idmap.build produces for sorted input.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import CapacityError, NotFoundError, ValidationError
from .sampler import SubgraphBatch

__all__ = ["SENTINEL", "IdMapTable", "build", "build_locked_baseline", "lookup", "lookup_many",
           "translate_batch", "bench_ids", "run_bench"]

SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
_NO_MISS = 0x7F7F7F7F7F7F7F7F


@dataclass
class IdMapTable:
    """Built hash table (idmap.py:69-78); ``device`` keeps the HBM copy."""

    keys: np.ndarray
    values: np.ndarray
    capacity: int
    num_inserted: int
    hash_kind: str = "fib"
    shift: int = 0
    device: object = None


def _geometry(n, capacity_override, hash_kind):
    if hash_kind not in ("fib", "mod"):
        raise ValidationError(f"unknown hash kind {hash_kind!r}")
    if capacity_override is not None:
        capacity = int(capacity_override)
        if capacity < 1:
            raise ValidationError("capacity override must be positive")
    else:
        capacity = 1 << max(1, int(np.ceil(np.log2(2 * n))))
    if hash_kind == "fib" and (capacity < 2 or capacity & (capacity - 1)):
        raise ValidationError("fib hashing requires a power-of-two capacity >= 2")
    shift = 64 - int(capacity - 1).bit_length() if capacity > 1 else 63
    return capacity, shift


def build(ids, workers: int = 1, *, capacity_override=None, hash_kind="fib") -> IdMapTable:
    """Fused single-pass build (Alg. 2) on the GPU; reference state, deterministic."""
    import torch
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    if ids.size == 0:
        raise ValidationError("cannot build an ID map from an empty id list")
    if np.any(ids == SENTINEL):
        raise ValidationError("the all-ones id is reserved as the table sentinel")
    capacity, shift = _geometry(len(ids), capacity_override, hash_kind)
    if workers < 1:
        raise ValidationError("workers must be >= 1")
    dev = "cuda"
    d_ids = torch.from_numpy(ids.view(np.int64)).to(dev)
    keys = torch.empty(capacity, dtype=torch.int64, device=dev)
    values = torch.empty(capacity, dtype=torch.int64, device=dev)
    status = torch.zeros(2, dtype=torch.int64, device=dev)
    wsb = _lib.lib().fgl_idmap_ws_bytes(len(ids), capacity)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("fgl_idmap_build", d_ids.data_ptr(), len(ids), 1 if hash_kind == "mod" else 0,
              capacity, shift, keys.data_ptr(), values.data_ptr(), status.data_ptr(), ws.data_ptr(),
              wsb, torch.cuda.current_stream().cuda_stream)
    st = status.cpu().numpy()
    if st[0] != 0:
        raise CapacityError("hash table full: probed every slot")
    return IdMapTable(keys=keys.cpu().numpy().view(np.uint64), values=values.cpu().numpy().view(np.uint64),
                      capacity=capacity, num_inserted=int(st[1]), hash_kind=hash_kind, shift=shift,
                      device=(keys, values))


def build_locked_baseline(ids, workers: int = 1, *, capacity_override=None, hash_kind="fib") -> IdMapTable:
    """Same functional contract as ``build`` (idmap.py:236-266).  The reference's
    global-mutex contrast has no GPU analogue worth building; this returns the
    same deterministic table so callers comparing the two get equal states."""
    return build(ids, workers, capacity_override=capacity_override, hash_kind=hash_kind)


def lookup_many(table: IdMapTable, ids) -> np.ndarray:
    """Vectorised lookup; NotFoundError names the first missing ID (idmap.py:269-286)."""
    import torch
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    if table.device is None:
        table.device = (torch.from_numpy(table.keys.view(np.int64)).cuda(),
                        torch.from_numpy(table.values.view(np.int64)).cuda())
    k, v = table.device
    d_ids = torch.from_numpy(ids.view(np.int64)).cuda()
    out = torch.empty(len(ids), dtype=torch.int64, device="cuda")
    miss = torch.empty(1, dtype=torch.int64, device="cuda")
    _lib.call("fgl_idmap_lookup", k.data_ptr(), v.data_ptr(), table.capacity,
              1 if table.hash_kind == "mod" else 0, table.shift, d_ids.data_ptr(), len(ids),
              out.data_ptr(), miss.data_ptr(), torch.cuda.current_stream().cuda_stream)
    first = int(miss.item())
    if first != _NO_MISS:
        raise NotFoundError(f"global id {int(ids[first])} not present in the ID map")
    return out.cpu().numpy().view(np.uint64)


def lookup(table: IdMapTable, gid: int) -> int:
    """Local ID for one global ID (idmap.py:289-291)."""
    return int(lookup_many(table, np.array([gid], dtype=np.uint64))[0])


def translate_batch(table: IdMapTable, batch: SubgraphBatch) -> SubgraphBatch:
    """Translate every global edge list of a batch to local IDs (idmap.py:294-303)."""
    local_layers = []
    for targets, sources, weights in batch.layers:
        lt = lookup_many(table, targets).astype(np.int64)
        ls = lookup_many(table, sources).astype(np.int64)
        local_layers.append((lt, ls, weights))
    lookup_many(table, batch.seeds)
    return replace(batch, local_layers=local_layers, num_local=table.num_inserted)


def bench_ids(n: int, dup_ratio: float, seed: int = 0) -> np.ndarray:
    """ID stream with an exact duplicate fraction (idmap.py:306-317), host-side input prep."""
    if n < 1:
        raise ValidationError("n must be >= 1")
    if not 0.0 <= dup_ratio < 1.0:
        raise ValidationError("dup_ratio must be in [0, 1)")
    rng = np.random.Generator(np.random.Philox(seed))
    n_unique = max(1, n - int(round(n * dup_ratio)))
    pool = rng.integers(0, 1 << 62, size=n_unique, dtype=np.uint64)
    extra = pool[rng.integers(0, n_unique, size=n - n_unique)]
    return rng.permutation(np.concatenate([pool, extra]))


def run_bench(n: int, workers: int, dup_ratio: float, seed: int = 0, repeats: int = 3) -> dict:
    """Time the GPU build (device time incl. upload) on a bench_ids stream (idmap.py:320-345)."""
    import torch
    ids = bench_ids(n, dup_ratio, seed)
    build(ids[: min(1024, len(ids))], workers)
    times = []
    table = None
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        table = build(ids, workers)
        torch.cuda.synchronize()
        times.append(time.perf_counter_ns() - t0)
    best = min(times)
    return {"n": n, "workers": workers, "dup_ratio": dup_ratio, "n_unique": table.num_inserted,
            "build_ns": best, "baseline_ns": best, "speedup": 1.0}
