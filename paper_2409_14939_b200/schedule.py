"""Match-Reorder scheduling: drop-in for ``minigl.schedule``.

Set intersections run on the GPU over node bitmaps (fgl_mark_bitmaps +
fgl_match_counts for all pairs of a window in one pass, fgl_bitmap_test for a
transition's overlap/load split); the greedy chain itself is a tiny n x n
host loop with the reference's tie rules (schedule.py:92-113).  In the
trainer the bitmaps come straight from the window sampler and the load set
is never materialised: the loader tests membership per row.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ValidationError
from .sampler import SubgraphBatch

__all__ = ["MatchMatrix", "Transition", "BatchSchedule", "match_degree", "build_match_matrix",
           "greedy_reorder", "compute_transition", "schedule_window", "match_stats"]


@dataclass
class MatchMatrix:
    n: int
    m: np.ndarray


@dataclass
class Transition:
    overlap_ids: np.ndarray
    load_ids: np.ndarray


@dataclass
class BatchSchedule:
    order: list
    transitions: list
    window_traffic_bytes: int
    batch_nodes: list
    feature_dim: int


def _unique_ids(batch_or_ids) -> np.ndarray:
    if isinstance(batch_or_ids, SubgraphBatch) or hasattr(batch_or_ids, "unique_nodes"):
        return np.asarray(batch_or_ids.unique_nodes, dtype=np.uint64)
    return np.unique(np.asarray(batch_or_ids, dtype=np.uint64))


def _bitmaps(sets):
    """Device bitmaps of a list of sorted ID sets (IDs < 2^31)."""
    import torch
    top = max((int(s[-1]) for s in sets if len(s)), default=0)
    if top >= 2**31:
        raise ValidationError("device match-degree path needs node IDs < 2^31")
    words = (top >> 5) + 1
    words = (words + 3) // 4 * 4
    off = np.zeros(len(sets) + 1, dtype=np.int64)
    np.cumsum([len(s) for s in sets], out=off[1:])
    flat = np.concatenate(sets).astype(np.int32) if off[-1] else np.zeros(1, np.int32)
    ids = torch.from_numpy(flat).cuda()
    d_off = torch.from_numpy(off).cuda()
    bm = torch.empty(len(sets) * words, dtype=torch.int32, device="cuda")
    _lib.call("fgl_mark_bitmaps", ids.data_ptr(), d_off.data_ptr(), len(sets), int(off[-1]), words,
              bm.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return bm, words


def _pair_counts(sets) -> np.ndarray:
    """|a ∩ b| for all pairs, on the GPU (<= 16 sets per call, chunked beyond)."""
    import torch
    n = len(sets)
    out = np.zeros((n, n), dtype=np.int64)
    bm, words = _bitmaps(sets)
    pairs = torch.zeros(120, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    groups = [list(range(i, min(i + 8, n))) for i in range(0, n, 8)]
    for gi, ga in enumerate(groups):
        for gb in groups[gi:]:
            idx = ga if ga == gb else ga + gb
            sub = torch.cat([bm[i * words : (i + 1) * words] for i in idx])
            if len(idx) < 2:
                continue
            _lib.call("fgl_match_counts", sub.data_ptr(), words, len(idx), pairs.data_ptr(), st)
            p = pairs.cpu().numpy()
            for a in range(len(idx)):
                for b in range(a + 1, len(idx)):
                    k = a * 16 - a * (a + 1) // 2 + (b - a - 1)
                    out[idx[a], idx[b]] = out[idx[b], idx[a]] = int(p[k])
    return out


def match_degree(a, b) -> float:
    """|a ∩ b| / min(|a|, |b|) (schedule.py:68-75)."""
    a = _unique_ids(a)
    b = _unique_ids(b)
    if a.size == 0 or b.size == 0:
        raise ValidationError("match degree is undefined for empty node sets")
    return int(_pair_counts([a, b])[0, 1]) / min(len(a), len(b))


def build_match_matrix(batches) -> MatchMatrix:
    """All-pairs match degrees, zero diagonal (schedule.py:78-89)."""
    n = len(batches)
    if n < 2:
        raise ValidationError("need at least two batches for a match matrix")
    ids = [_unique_ids(b) for b in batches]
    if any(len(s) == 0 for s in ids):
        raise ValidationError("match degree is undefined for empty node sets")
    cnt = _pair_counts(ids)
    sizes = np.array([len(s) for s in ids], dtype=np.int64)
    m = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1, n):
            m[i, j] = m[j, i] = int(cnt[i, j]) / int(min(sizes[i], sizes[j]))
    return MatchMatrix(n=n, m=m)


def greedy_reorder(matrix: MatchMatrix) -> list:
    """Greedy chain from batch 0; ties and non-positive rows -> lowest index."""
    from .trainer import greedy_order
    if matrix.n < 1:
        raise ValidationError("empty match matrix")
    return greedy_order(matrix.m)


def compute_transition(prev, nxt):
    """(overlap, load) node sets of a transition (schedule.py:116-123)."""
    import torch
    prev_ids = _unique_ids(prev)
    next_ids = _unique_ids(nxt)
    if len(next_ids) == 0:
        return next_ids.copy(), next_ids.copy()
    top = max(int(next_ids[-1]), int(prev_ids[-1]) if len(prev_ids) else 0)
    words = ((top >> 5) + 1 + 3) // 4 * 4
    bm, _ = _bitmaps([prev_ids if len(prev_ids) else np.zeros(0, np.uint64), np.array([top], np.uint64)])
    hit = torch.empty(len(next_ids), dtype=torch.int8, device="cuda")
    nx = torch.from_numpy(next_ids.astype(np.int32)).cuda()
    _lib.call("fgl_bitmap_test", nx.data_ptr(), len(next_ids), bm.data_ptr(), hit.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    h = hit.cpu().numpy().astype(bool)
    del words
    return next_ids[h], next_ids[~h]


def schedule_window(batches, enable_reorder: bool, feature_dim: int) -> BatchSchedule:
    """Order a window and account its host-to-device traffic (schedule.py:126-155)."""
    n = len(batches)
    if n < 1:
        raise ValidationError("window must contain at least one batch")
    if feature_dim < 1:
        raise ValidationError("feature_dim must be >= 1")
    order = greedy_reorder(build_match_matrix(batches)) if (enable_reorder and n >= 2) else list(range(n))
    executed = [batches[i] for i in order]
    nodes = [_unique_ids(b) for b in executed]
    transitions = []
    loaded = len(nodes[0])
    for prev, nxt in zip(nodes, nodes[1:]):
        ov, ld = compute_transition(prev, nxt)
        transitions.append(Transition(overlap_ids=ov, load_ids=ld))
        loaded += len(ld)
    return BatchSchedule(order=order, transitions=transitions,
                         window_traffic_bytes=4 * feature_dim * loaded, batch_nodes=nodes,
                         feature_dim=feature_dim)


def match_stats(batches) -> dict:
    """Mean off-diagonal match degree and its spread (schedule.py:158-167)."""
    m = build_match_matrix(batches)
    iu = np.triu_indices(m.n, k=1)
    pairs = m.m[iu]
    return {"avg_match_degree": float(pairs.mean()), "delta_match": float(pairs.max() - pairs.min()),
            "num_batches": m.n}
