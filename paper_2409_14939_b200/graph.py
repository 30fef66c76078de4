"""Graph input contract and its device-resident copy.

The drop-in functions accept the reference's own ``minigl.graph.Graph``
(graph.py:25-87) or :class:`Graph` below -- anything with ``num_nodes``,
``row_offsets`` (uint64[N+1]), ``col_indices`` (uint64[E]) and optional
``edge_weights`` (f32[E]).  :func:`device_graph` uploads the forward CSR once
per graph object (int64 offsets, int32 columns) and caches it.

Graph construction itself is out of scope for the hot path (SURVEY.md
section 2, "construction stays host-side"); :func:`chung_lu_graph` is a fast
seeded generator used by bench.py to build the large BASELINE shapes that the
reference's per-node Python generator (graph.py:250-276) cannot reach.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(eq=False)
class Graph:
    """Host CSR with the reference's field names (forward adjacency only is
    required by the sampler; the transpose is optional here)."""

    num_nodes: int
    num_edges: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    edge_weights: np.ndarray | None = None
    t_row_offsets: np.ndarray | None = None
    t_col_indices: np.ndarray | None = None

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets.astype(np.int64))


@dataclass(eq=False)
class FeatureMatrix:
    """Dense row-major float32 node features (graph.py:90-114)."""

    num_nodes: int
    dim: int
    data: np.ndarray

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float32)
        if self.data.shape != (self.num_nodes, self.dim):
            raise ValidationError(
                f"feature data shape {self.data.shape} != ({self.num_nodes}, {self.dim})")


class DeviceGraph:
    """Forward CSR resident in HBM: int64 row offsets, int32 columns, f32 weights."""

    def __init__(self, num_nodes, row_offsets, col_indices, edge_weights=None):
        from . import _lib
        self.num_nodes = int(num_nodes)
        self.row_offsets = row_offsets
        self.col_indices = col_indices
        self.edge_weights = edge_weights
        self.num_edges = int(col_indices.numel())
        self._struct = _lib.FglGraph(
            self.num_nodes, self.num_edges, row_offsets.data_ptr(), col_indices.data_ptr(),
            edge_weights.data_ptr() if edge_weights is not None else None)

    @property
    def struct(self):
        return self._struct

    @classmethod
    def from_host(cls, g, device="cuda"):
        import torch
        n = int(g.num_nodes)
        if n < 1:
            raise ValidationError("graph must have at least one node")
        if n >= 2**31:
            raise ValidationError("device graphs use int32 node IDs (num_nodes < 2^31)")
        off = torch.from_numpy(np.ascontiguousarray(g.row_offsets).astype(np.int64, copy=False))
        col = torch.from_numpy(np.ascontiguousarray(g.col_indices).astype(np.int32))
        w = getattr(g, "edge_weights", None)
        wt = None if w is None else torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32))
        return cls(n, off.to(device), col.to(device), None if wt is None else wt.to(device))


_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def device_graph(g, device="cuda") -> DeviceGraph:
    """Upload (once, cached per host graph object) and return the device CSR."""
    if isinstance(g, DeviceGraph):
        return g
    try:
        dg = _cache.get(g)
    except TypeError:
        dg = None
    if dg is None:
        dg = DeviceGraph.from_host(g, device)
        try:
            _cache[g] = dg
        except TypeError:
            pass
    return dg


def chung_lu_graph(num_nodes: int, num_edges: int, exponent: float = 2.3, seed: int = 0,
                   device="cuda", permute: bool = True) -> DeviceGraph:
    """Seeded Chung-Lu power-law graph built on the GPU with torch ops.

    Expected degree of node i is proportional to (i+1)^(-1/(exponent-1)).
    ``num_edges/2`` endpoint pairs are drawn by inverse-CDF sampling, stored in
    both directions (undirected, like the reference generator), self loops and
    duplicate pairs removed, node IDs randomly permuted, and packed into the
    canonical (src, dst)-sorted CSR of graph.py:151-183.  Input preparation
    only -- not part of the timed hot path.
    """
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    n = int(num_nodes)
    a = 1.0 / (exponent - 1.0)
    w = torch.arange(1, n + 1, device=device, dtype=torch.float64).pow_(-a)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    perm = torch.randperm(n, device=device, generator=g) if permute else None
    want_pairs = int(num_edges) // 2
    pairs = torch.empty(0, dtype=torch.int64, device=device)
    draw = int(want_pairs * 1.1) + 16
    for _ in range(64):  # top up until enough distinct undirected pairs exist
        parts = []
        chunk = 1 << 25
        for i in range(0, draw, chunk):
            m = min(chunk, draw - i)
            u = torch.rand(m, 2, device=device, dtype=torch.float64, generator=g)
            parts.append(torch.searchsorted(cdf, u).clamp_(max=n - 1))
        ends = torch.cat(parts)
        if perm is not None:
            ends = perm[ends]
        s, d = ends[:, 0], ends[:, 1]
        keep = s != d
        s, d = s[keep], d[keep]
        lo = torch.minimum(s, d) * n + torch.maximum(s, d)
        pairs = torch.unique(torch.cat([pairs, lo]))
        if pairs.numel() >= want_pairs:
            break
        draw = int((want_pairs - pairs.numel()) * 1.5) + 1024
    if pairs.numel() > want_pairs:  # keep a seeded random subset of exactly want_pairs
        pick = torch.randperm(pairs.numel(), device=device, generator=g)[:want_pairs]
        pairs = pairs[pick]
    u, v = pairs // n, pairs % n
    key = torch.sort(torch.cat([u * n + v, v * n + u])).values  # both directions, (src, dst) order
    src = key // n
    col = (key % n).to(torch.int32)
    counts = torch.bincount(src, minlength=n)
    off = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    return DeviceGraph(n, off, col.contiguous(), None)


def to_host(dg: DeviceGraph) -> Graph:
    """Host (uint64) copy of a device graph, e.g. for the CPU baseline."""
    off = dg.row_offsets.cpu().numpy().astype(np.uint64)
    col = dg.col_indices.cpu().numpy().astype(np.uint64)
    w = None if dg.edge_weights is None else dg.edge_weights.cpu().numpy()
    return Graph(dg.num_nodes, dg.num_edges, off, col, w)
