"""numpy restatement of the reference hot path (oracle -- test infrastructure only).

Every function cites the reference (``/root/reference``) file:line whose
behaviour it restates; bare module names mean ``pkg/src/minigl/<name>``.
The restatement is written for clarity and vectorised numpy speed, not as a
copy of the reference's code; ``tests/test_oracle_golden.py`` pins it to the
reference's own outputs (``tests/golden``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import philox

U64 = np.uint64
SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
FIB = np.uint64(0x9E3779B97F4A7C15)

__all__ = [
    "SENTINEL", "CSRGraph", "graph_from_edges", "gen_power_law", "derive_seed",
    "Batch", "sample_khop", "sample_random_walk", "epoch_seed_batches", "IdTable", "idmap_build",
    "idmap_lookup", "layer_edge_weights", "edges_to_csr", "csr_transpose",
    "prepare_batch", "tile_plan_error", "aggregate", "dense", "softmax_xent",
    "init_params", "forward", "backward", "sgd_step", "match_matrix",
    "greedy_order", "window_schedule", "epoch_h2d_bytes", "cache_mask", "train_split",
    "train", "train_step", "evaluate_params", "two_cluster_task",
]


# ---------------------------------------------------------------- seeds -----

def derive_seed(base: int, *parts: int) -> int:
    """Child seed of (base, *parts): first SeedSequence word (``trainer.py:40-42``)."""
    return int(np.random.SeedSequence((base, *parts)).generate_state(1)[0])


# ---------------------------------------------------------------- graph -----

@dataclass(eq=False)
class CSRGraph:
    """Forward + transposed uint64 CSR, optional f32 weights (``graph.py:25-87``)."""

    num_nodes: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    t_row_offsets: np.ndarray
    t_col_indices: np.ndarray
    edge_weights: np.ndarray | None = None
    t_edge_weights: np.ndarray | None = None

    @property
    def num_edges(self) -> int:
        return int(self.row_offsets[-1])


def _offsets(n, rows_sorted):
    counts = np.bincount(rows_sorted.astype(np.int64), minlength=n)
    out = np.zeros(n + 1, dtype=U64)
    out[1:] = np.cumsum(counts).astype(U64)
    return out


def graph_from_edges(n, src, dst, weights=None) -> CSRGraph:
    """Canonical (src, dst)-lexicographic CSR plus its transpose (``graph.py:151-183``).

    Duplicate edges keep their input order (stable sorts on both sides).
    """
    src = np.asarray(src, dtype=U64)
    dst = np.asarray(dst, dtype=U64)
    w = None if weights is None else np.asarray(weights, dtype=np.float32)
    fwd = np.lexsort((dst, src))
    s1, d1 = src[fwd], dst[fwd]
    w1 = None if w is None else w[fwd]
    rev = np.lexsort((s1, d1))
    return CSRGraph(
        num_nodes=int(n),
        row_offsets=_offsets(n, s1),
        col_indices=d1.copy(),
        t_row_offsets=_offsets(n, d1[rev]),
        t_col_indices=s1[rev].copy(),
        edge_weights=w1,
        t_edge_weights=None if w1 is None else w1[rev],
    )


def gen_power_law(n: int, avg_degree: float, seed: int) -> CSRGraph:
    """Preferential-attachment generator of ``graph.py:225-233`` / ``:250-276``.

    m = round(avg_degree / 2) endpoints are drawn per new node from the running
    endpoint multiset; the distinct picks become undirected edges stored in
    both directions.  Deterministic under ``Generator(Philox(seed))``.
    """
    rng = np.random.Generator(np.random.Philox(seed))
    m = max(1, round(avg_degree / 2))
    if n <= m:
        raise ValueError("num_nodes must exceed avg_degree/2")
    pool = np.empty(4 * m * n, dtype=np.int64)
    src_parts, dst_parts = [], []
    first = np.arange(1, m + 1, dtype=np.int64)
    src_parts.append(np.zeros(m, dtype=np.int64))
    dst_parts.append(first)
    pool[:m] = 0
    pool[m : 2 * m] = first
    used = 2 * m
    for node in range(m + 1, n):
        chosen = np.unique(pool[rng.integers(0, used, size=m)])
        k = len(chosen)
        src_parts.append(np.full(k, node, dtype=np.int64))
        dst_parts.append(chosen)
        pool[used : used + k] = node
        pool[used + k : used + 2 * k] = chosen
        used += 2 * k
    a = np.concatenate(src_parts)
    b = np.concatenate(dst_parts)
    return graph_from_edges(n, np.concatenate([a, b]), np.concatenate([b, a]))


# -------------------------------------------------------------- sampler -----

@dataclass
class Batch:
    """Sampled batch in global IDs (``sampler.py:47-68``)."""

    seeds: np.ndarray
    layers: list  # [(targets u64, sources u64, weights f32)]
    unique_nodes: np.ndarray
    draws: int = 0  # Philox draws consumed (candidates over all hops)

    def num_sampled_edges(self) -> int:
        return sum(len(t) for t, _, _ in self.layers)


def sample_khop(g: CSRGraph, seeds, fanouts, seed: int) -> Batch:
    """K-hop uniform sampling (``sampler.py:86-139``), keys from the Philox stream.

    Per hop: frontier = sorted distinct IDs; one draw per candidate out-edge in
    frontier-major CSR order at consecutive stream positions; each frontier
    node keeps its min(deg, fanout) smallest (key, edge-slot) pairs, emitted in
    ascending key order.  No draws are consumed by an edgeless hop.
    """
    seeds = np.asarray(seeds, dtype=U64)
    if seeds.size == 0 or int(seeds.max()) >= g.num_nodes:
        raise ValueError("bad seeds")
    key = philox.key_for_seed(seed)
    off = g.row_offsets.astype(np.int64)
    pos = 0
    frontier = np.unique(seeds)
    layers, seen = [], [seeds]
    for fan in fanouts:
        f_idx = frontier.astype(np.int64)
        lo, deg = off[f_idx], off[f_idx + 1] - off[f_idx]
        total = int(deg.sum())
        if total == 0:
            e = np.empty(0, dtype=U64)
            layers.append((e, e.copy(), np.empty(0, dtype=np.float32)))
            frontier = e
            continue
        k53 = philox.keys53(key, pos, total)
        pos += total
        node = np.repeat(np.arange(len(frontier)), deg)
        seg_start = np.repeat(np.cumsum(deg) - deg, deg)
        slot = np.arange(total) - seg_start
        # sort by node, then key, then slot (lexsort: last key is primary)
        perm = np.lexsort((slot, k53, node))
        keep = perm[(np.arange(total) - seg_start) < fan]  # rank within node < fanout
        edge = lo[node[keep]] + slot[keep]
        tgt = frontier[node[keep]]
        src = g.col_indices[edge]
        w = (g.edge_weights[edge] if g.edge_weights is not None
             else np.ones(len(edge), dtype=np.float32))
        layers.append((tgt, src, w))
        seen += [tgt, src]
        frontier = np.unique(src)
    return Batch(seeds=seeds, layers=layers, unique_nodes=np.unique(np.concatenate(seen)),
                 draws=pos)


def sample_random_walk(g: CSRGraph, seeds, length: int, seed: int) -> Batch:
    """Uniform random walk (``sampler.py:142-186``): at each step the alive
    walkers whose node has out-degree > 0, in seed order, take consecutive
    draws u of the Philox(seed) stream and move to
    col[off[v] + floor(u * deg)] (float64 product, truncation); a sink ends
    its walk without a draw.  Edges step-major; unique over seeds, targets and
    sources."""
    seeds = np.asarray(seeds, dtype=U64)
    if seeds.size == 0 or int(seeds.max()) >= g.num_nodes:
        raise ValueError("bad seeds")
    if length < 1:
        raise ValueError("walk length must be >= 1")
    key = philox.key_for_seed(seed)
    off = g.row_offsets.astype(np.int64)
    cur = seeds.astype(np.int64).copy()
    alive = np.ones(len(seeds), dtype=bool)
    pos = 0
    ts, ss, ws = [], [], []
    for _ in range(length):
        idx = np.flatnonzero(alive)
        if idx.size == 0:
            break
        deg = off[cur[idx] + 1] - off[cur[idx]]
        alive[idx[deg == 0]] = False
        idx = idx[deg > 0]
        deg = deg[deg > 0]
        if idx.size == 0:
            break
        u = philox.keys53(key, pos, len(idx)).astype(np.float64) * 2.0 ** -53
        pos += len(idx)
        edge = off[cur[idx]] + (u * deg).astype(np.int64)
        nxt = g.col_indices[edge].astype(np.int64)
        ts.append(cur[idx].astype(U64))
        ss.append(nxt.astype(U64))
        ws.append(g.edge_weights[edge] if g.edge_weights is not None else np.ones(len(idx), dtype=np.float32))
        cur[idx] = nxt
    t = np.concatenate(ts) if ts else np.empty(0, dtype=U64)
    s = np.concatenate(ss) if ss else np.empty(0, dtype=U64)
    w = np.concatenate(ws) if ws else np.empty(0, dtype=np.float32)
    return Batch(seeds=seeds, layers=[(t, s, w)], unique_nodes=np.unique(np.concatenate([seeds, t, s])),
                 draws=pos)


def epoch_seed_batches(train_ids, batch_size: int, shuffle_seed: int):
    """Philox permutation split into batches (``sampler.py:189-198``)."""
    perm = np.random.Generator(np.random.Philox(shuffle_seed)).permutation(
        np.asarray(train_ids, dtype=U64))
    return [perm[i : i + batch_size] for i in range(0, len(perm), batch_size)]


# ---------------------------------------------------------------- idmap -----

@dataclass
class IdTable:
    """Open-addressing table state (``idmap.py:69-78``)."""

    keys: np.ndarray
    values: np.ndarray
    capacity: int
    num_inserted: int
    hash_kind: str
    shift: int


def _table_geometry(n, capacity_override, hash_kind):
    # idmap.py:175-195: capacity = smallest power of two >= 2n (>= 2)
    cap = int(capacity_override) if capacity_override is not None else 1 << max(1, (2 * n - 1).bit_length())
    shift = 64 - (cap - 1).bit_length() if cap > 1 else 63
    return cap, shift


def _home(gid: int, cap: int, shift: int, hash_kind: str) -> int:
    if hash_kind == "mod":
        return gid % cap
    return ((gid * int(FIB)) & 0xFFFFFFFFFFFFFFFF) >> shift


def idmap_build(ids, *, capacity_override=None, hash_kind="fib") -> IdTable:
    """Single-worker Fused-Map build (``idmap.py:88-117``, ``:198-233``, workers=1).

    Sequential linear probing from the hash slot; a new key takes the first
    empty slot and the next local ID (first-seen order); duplicates are no-ops.
    """
    ids = [int(x) for x in np.asarray(ids, dtype=U64)]
    cap, shift = _table_geometry(len(ids), capacity_override, hash_kind)
    keys = np.full(cap, SENTINEL, dtype=U64)
    vals = np.zeros(cap, dtype=U64)
    nxt = 0
    sent = int(SENTINEL)
    for gid in ids:
        s = _home(gid, cap, shift, hash_kind)
        for _ in range(cap):
            k = int(keys[s])
            if k == gid:
                break
            if k == sent:
                keys[s] = gid
                vals[s] = nxt
                nxt += 1
                break
            s = s + 1 if s + 1 < cap else 0
        else:
            raise OverflowError("hash table full")
    return IdTable(keys, vals, cap, nxt, hash_kind, shift)


def idmap_lookup(t: IdTable, ids) -> np.ndarray:
    """Probe lookup; raises KeyError(first missing gid) (``idmap.py:154-172``, ``:269-286``)."""
    out = np.empty(len(ids), dtype=U64)
    sent = int(SENTINEL)
    for i, gid in enumerate(int(x) for x in np.asarray(ids, dtype=U64)):
        s = _home(gid, t.capacity, t.shift, t.hash_kind)
        for _ in range(t.capacity):
            k = int(t.keys[s])
            if k == gid:
                out[i] = t.values[s]
                break
            if k == sent:
                raise KeyError(gid)
            s = s + 1 if s + 1 < t.capacity else 0
        else:
            raise KeyError(gid)
    return out


# -------------------------------------------------------------- compute -----

def layer_edge_weights(arch, lt, ls, n):
    """GCN 1/sqrt(indeg_t * outdeg_s) over per-hop local degrees, fp64 -> f32;
    GIN unit weights (``trainer.py:156-162``).  "sage" (EXTENSION, SURVEY
    8(c): the reference has no GraphSAGE; oracle = this restatement): mean
    aggregation 1/indeg_t in fp64 -> f32, with the GIN-style root term added
    in forward / backward."""
    if arch == "gin":
        return np.ones(len(lt), dtype=np.float32)
    if arch == "sage":
        indeg = np.bincount(lt, minlength=n).astype(np.int64)
        return (1.0 / indeg[lt].astype(np.float64)).astype(np.float32)
    indeg = np.bincount(lt, minlength=n).astype(np.int64)
    outdeg = np.bincount(ls, minlength=n).astype(np.int64)
    prod = (indeg[lt] * outdeg[ls]).astype(np.float64)
    return (1.0 / np.sqrt(prod)).astype(np.float32)


def edges_to_csr(n, targets, sources, weights):
    """Stable pack by target (``compute.py:219-230``)."""
    t = np.asarray(targets, dtype=np.int64)
    perm = np.argsort(t, kind="stable")
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(np.bincount(t, minlength=n))
    return (indptr, np.asarray(sources, dtype=np.int64)[perm],
            np.asarray(weights, dtype=np.float32)[perm])


def csr_transpose(indptr, indices, weights, ncols):
    """Exact transpose, weights travel with edges, stable by source (``compute.py:233-239``)."""
    rows = np.repeat(np.arange(len(indptr) - 1, dtype=np.int64), np.diff(indptr))
    return edges_to_csr(ncols, indices, rows, weights)


def prepare_batch(b: Batch, arch: str = "gcn"):
    """Local-ID translation + per-model-layer CSR/transposes (``trainer.py:165-179``).

    Trainer path (map_workers=1 over sorted unique IDs): local ID = rank of the
    global ID in ``unique_nodes``.  Model layer i consumes hop k-1-i.
    Returns (local_layers, seed_locals, n, csr_layers).
    """
    uniq = b.unique_nodes
    n = len(uniq)
    loc = lambda a: np.searchsorted(uniq, np.asarray(a, dtype=U64)).astype(np.int64)
    local_layers = [(loc(t), loc(s), w) for t, s, w in b.layers]
    seed_locals = loc(b.seeds)
    csr = []
    for lt, ls, _ in reversed(local_layers):
        w = layer_edge_weights(arch, lt, ls, n)
        ip, ix, cw = edges_to_csr(n, lt, ls, w)
        csr.append((ip, ix, cw) + csr_transpose(ip, ix, cw, n))
    return local_layers, seed_locals, n, csr


def tile_plan_error(num_targets, dim, row_lengths, x=8, y=32, scratch=128 * 1024):
    """None if ``plan_tiles`` accepts the shape, else the reason (``compute.py:34-112``)."""
    if x < 1 or y < 1:
        return "tile dims"
    if x * y >= 1024:
        return "cells"
    if scratch < 1:
        return "scratch"
    rl = np.asarray(row_lengths, dtype=np.int64)
    for g0 in range(0, num_targets, x):
        mf = int(rl[g0 : g0 + x].max()) if g0 < num_targets else 0
        if 4 * x * y + 4 * x * mf > scratch:
            return f"group {g0}"
    return None


def aggregate(indptr, indices, weights, feats):
    """h_u = sum_e w_e * x_{idx_e}: fp32 product then fp32 add per edge, in CSR
    order, no FMA (``compute.py:115-148``).  Empty rows are exactly zero."""
    indptr = np.asarray(indptr, dtype=np.int64)
    feats = np.asarray(feats, dtype=np.float32)
    n = len(indptr) - 1
    out = np.zeros((n, feats.shape[1]), dtype=np.float32)
    deg = np.diff(indptr)
    if n == 0 or deg.max(initial=0) == 0:
        return out
    order = np.argsort(-deg, kind="stable")  # rows with more than k edges form a prefix
    asc = deg[order][::-1]
    weights = np.asarray(weights, dtype=np.float32)
    indices = np.asarray(indices, dtype=np.int64)
    for k in range(int(asc[-1])):
        rows = order[: n - int(np.searchsorted(asc, k, side="right"))]
        e = indptr[rows] + k
        out[rows] = out[rows] + weights[e][:, None] * feats[indices[e]]
    return out


def dense(h, w, b=None, relu=False):
    """act(h @ W + b) in fp32 (``compute.py:198-216``)."""
    z = np.asarray(h, dtype=np.float32) @ np.asarray(w, dtype=np.float32)
    if b is not None:
        z = z + np.asarray(b, dtype=np.float32)
    return np.maximum(z, 0.0) if relu else z


def softmax_xent(logits, labels):
    """Mean CE in float64; dlogits = (p - onehot)/B as f32 (``trainer.py:198-209``)."""
    z = np.asarray(logits, dtype=np.float64)
    z = z - z.max(axis=1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    rows = np.arange(len(labels))
    loss = float(-np.log(p[rows, labels] + 1e-30).mean())
    p[rows, labels] -= 1.0
    return loss, (p / len(labels)).astype(np.float32)


def init_params(layer_dims, seed):
    """Glorot-normal weights, zero biases (``trainer.py:145-153``)."""
    rng = np.random.Generator(np.random.Philox(derive_seed(seed, 101)))
    out = []
    for a, c in zip(layer_dims[:-1], layer_dims[1:]):
        w = (rng.standard_normal((a, c)) * np.sqrt(2.0 / (a + c))).astype(np.float32)
        out.append([w, np.zeros(c, dtype=np.float32)])
    return out


def forward(x0, csr, params, arch="gcn"):
    """Per layer: aggregate, (+x for GIN), dense, ReLU except last (``trainer.py:182-195``)."""
    x, caches = x0, []
    last = len(params) - 1
    for i, ((ip, ix, cw, *_), (w, b)) in enumerate(zip(csr, params)):
        h = aggregate(ip, ix, cw, x)
        if arch in ("gin", "sage"):  # root / self term
            h = h + x
        z = dense(h, w, b)
        caches.append((x, h, z))
        x = z if i == last else np.maximum(z, 0.0)
    return x, caches


def backward(dout, caches, csr, params, arch="gcn"):
    """Reverse pass (``trainer.py:212-228``): dz, dW=h^T dz, db, dh=dz W^T,
    dx = aggregate over the transpose (+dh for GIN)."""
    grads = [None] * len(params)
    dx = dout
    for i in range(len(params) - 1, -1, -1):
        _, h, z = caches[i]
        dz = dx if i == len(params) - 1 else dx * (z > 0)
        grads[i] = [h.T @ dz, dz.sum(axis=0)]
        dh = dz @ params[i][0].T
        dx = aggregate(*csr[i][3:6], dh)
        if arch in ("gin", "sage"):
            dx = dx + dh
    return grads


def sgd_step(params, grads, lr):
    """In-place f32 SGD (``trainer.py:321-323``)."""
    for (w, b), (dw, db) in zip(params, grads):
        w -= lr * dw
        b -= lr * db


def train_step(b: Batch, feats, labels, params, lr, arch="gcn"):
    """One batch of the compute phase (``trainer.py:314-325``); returns (loss, grads)."""
    _, seed_locals, n, csr = prepare_batch(b, arch)
    x0 = np.asarray(feats)[b.unique_nodes.astype(np.int64)]
    out, caches = forward(x0, csr, params, arch)
    loss, dl = softmax_xent(out[seed_locals], np.asarray(labels)[b.seeds.astype(np.int64)])
    dout = np.zeros_like(out)
    dout[seed_locals] = dl
    grads = backward(dout, caches, csr, params, arch)
    sgd_step(params, grads, lr)
    return loss, grads


# ------------------------------------------------------------- schedule -----

def match_matrix(node_sets):
    """M_ij = |a∩b| / min(|a|,|b|), symmetric, zero diagonal (``schedule.py:68-89``)."""
    n = len(node_sets)
    m = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1, n):
            a, b = node_sets[i], node_sets[j]
            m[i, j] = m[j, i] = len(np.intersect1d(a, b, assume_unique=True)) / min(len(a), len(b))
    return m


def greedy_order(m):
    """Greedy chain from batch 0; argmax first max; non-positive -> lowest unused
    (``schedule.py:92-113``)."""
    n = len(m)
    order, used, cur = [0], {0}, 0
    for _ in range(n - 1):
        cand = [(m[cur, j] if j not in used else -1.0) for j in range(n)]
        best = int(np.argmax(cand))
        if cand[best] <= 0.0:
            best = min(j for j in range(n) if j not in used)
        order.append(best)
        used.add(best)
        cur = best
    return order


def window_schedule(node_sets, reorder: bool, dim: int):
    """Order + per-transition load sets + window bytes (``schedule.py:116-155``)."""
    n = len(node_sets)
    order = greedy_order(match_matrix(node_sets)) if (reorder and n >= 2) else list(range(n))
    ex = [node_sets[i] for i in order]
    loads = [ex[0]] + [np.setdiff1d(b, a, assume_unique=True) for a, b in zip(ex, ex[1:])]
    return order, ex, loads, 4 * dim * sum(len(x) for x in loads)


def cache_mask(num_nodes, cache_ratio, degrees):
    """Static-degree feature cache (``memsim.py:110-126``): the floor(ratio * N)
    highest-degree nodes, ties broken by lower node id."""
    mask = np.zeros(num_nodes, dtype=bool)
    k = int(np.floor(cache_ratio * num_nodes))
    if k > 0:
        ranked = np.lexsort((np.arange(num_nodes), -np.asarray(degrees).astype(np.int64)))
        mask[ranked[:k]] = True
    return mask


def epoch_h2d_bytes(windows_exec, windows_loads, dim, match=True, cached=None):
    """Host->device feature bytes of an epoch (``memsim.py:129-186``): Match reuse
    (batches after the first in a window load only their load set), then a
    static cache mask; returns (bytes_h2d, bytes_match, bytes_cache)."""
    h2d = mt = ch = 0
    for ex, loads in zip(windows_exec, windows_loads):
        for j, full in enumerate(ex):
            need = loads[j] if (match and j > 0) else full
            hit = int(cached[need.astype(np.int64)].sum()) if (cached is not None and len(need)) else 0
            h2d += (len(need) - hit) * 4 * dim
            mt += (len(full) - len(need)) * 4 * dim
            ch += hit * 4 * dim
    return h2d, mt, ch


# -------------------------------------------------------------- trainer -----

def train_split(num_nodes, seed):
    """80/20 Philox split (``trainer.py:273-278``)."""
    perm = np.random.Generator(np.random.Philox(derive_seed(seed, 7))).permutation(num_nodes).astype(U64)
    cut = max(1, int(0.8 * num_nodes))
    return perm[:cut], perm[cut:]


def train(g: CSRGraph, feats, labels, layer_dims, fanouts, *, arch="gcn", batch_size=64,
          window_n=8, epochs=1, lr=0.3, seed=0, reorder=True, match=True,
          train_ids=None, val_ids=None, evaluate=True):
    """Restated epoch driver (``trainer.py:246-349``) and evaluation (``:352-365``).

    Returns a list of per-epoch dicts {loss, accuracy, bytes_h2d, bytes_match}
    and the final params.
    """
    labels = np.asarray(labels, dtype=np.int64)
    feats = np.asarray(feats, dtype=np.float32)
    if train_ids is None or val_ids is None:
        tr, va = train_split(g.num_nodes, seed)
        train_ids = tr if train_ids is None else train_ids
        val_ids = va if val_ids is None else val_ids
    params = init_params(layer_dims, seed)
    seed_batches = epoch_seed_batches(train_ids, batch_size, derive_seed(seed, 11))
    windows = [seed_batches[i : i + window_n] for i in range(0, len(seed_batches), window_n)]
    report = []
    for _ in range(epochs):
        base = 0
        loss_sum, seen = 0.0, 0
        wex, wld = [], []
        for win in windows:
            sampled = [sample_khop(g, s, fanouts, derive_seed(seed, 13, base + j)) for j, s in enumerate(win)]
            base += len(win)
            order, ex, loads, _ = window_schedule([b.unique_nodes for b in sampled], reorder, feats.shape[1])
            wex.append(ex)
            wld.append(loads)
            for i in order:
                loss, _ = train_step(sampled[i], feats, labels, params, lr, arch)
                loss_sum += loss * len(sampled[i].seeds)
                seen += len(sampled[i].seeds)
        h2d, mt, _ = epoch_h2d_bytes(wex, wld, feats.shape[1], match=match)
        acc = evaluate_params(g, feats, labels, params, fanouts, batch_size, seed, val_ids, arch) \
            if (evaluate and len(val_ids)) else float("nan")
        report.append({"loss": loss_sum / max(seen, 1), "accuracy": acc,
                       "bytes_h2d": h2d, "bytes_match": mt})
    return report, params


def evaluate_params(g, feats, labels, params, fanouts, batch_size, seed, eval_ids, arch="gcn"):
    """Sampled-neighbourhood accuracy with fixed draws (``trainer.py:352-365``)."""
    correct = total = 0
    eval_ids = np.asarray(eval_ids, dtype=U64)
    for i in range(0, len(eval_ids), batch_size):
        s = eval_ids[i : i + batch_size]
        b = sample_khop(g, s, fanouts, derive_seed(seed, 17, i))
        _, seed_locals, _, csr = prepare_batch(b, arch)
        out, _ = forward(feats[b.unique_nodes.astype(np.int64)], csr, params, arch)
        correct += int((out[seed_locals].argmax(axis=1) == labels[s.astype(np.int64)]).sum())
        total += len(s)
    return correct / max(total, 1)


def two_cluster_task(num_nodes=200, dim=16, seed=0):
    """Synthetic two-cluster task (``trainer.py:379-410``) restated for test inputs."""
    rng = np.random.Generator(np.random.Philox(seed))
    half = num_nodes // 2
    labels = np.zeros(num_nodes, dtype=np.int64)
    labels[half:] = 1
    src, dst = [], []
    for u in range(num_nodes):
        lo, hi = (0, half) if u < half else (half, num_nodes)
        nb = lo + rng.integers(0, hi - lo, size=6)
        nb = nb[nb != u]
        src.append(np.full(len(nb), u))
        dst.append(nb)
        if rng.random() < 0.1:
            olo, ohi = (half, num_nodes) if u < half else (0, half)
            src.append(np.array([u]))
            dst.append(np.array([int(rng.integers(olo, ohi))]))
    s = np.concatenate(src)
    d = np.concatenate(dst)
    g = graph_from_edges(num_nodes, np.concatenate([s, d]), np.concatenate([d, s]))
    centers = rng.standard_normal((2, dim)) * 1.5
    x = rng.standard_normal((num_nodes, dim)).astype(np.float32)
    x += centers[labels].astype(np.float32)
    return g, x, labels
