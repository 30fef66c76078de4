"""Graph input contract and its device-resident copy.

The drop-in functions accept the reference's own ``minigl.graph.Graph``
(graph.py:25-87) or :class:`Graph` below -- anything with ``num_nodes``,
``row_offsets`` (uint64[N+1]), ``col_indices`` (uint64[E]) and optional
``edge_weights`` (f32[E]).  :func:`device_graph` uploads the forward CSR once
per graph object (int64 offsets, int32 columns) and caches it.

Input formats: :func:`from_edges` builds the CSR and
its transpose ON THE GPU with two stable counting sorts (fgl_stable_group),
bit-exact with the reference's lexsort-based from_edges (graph.py:151-183);
:func:`load_binary` / :func:`save_binary` read and write the reference's MGL1
format (graph.py:293-351; the file IO is host-side, a missing transpose is
rebuilt on the GPU).  :func:`chung_lu_graph` is a fast seeded generator used by
bench.py for the large BASELINE shapes the reference's per-node Python
generator (graph.py:250-276) cannot reach.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np

from .errors import MiniGLError, ValidationError


class FormatError(MiniGLError):
    """Malformed MGL1 file (graph.py FormatError)."""


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
    t_edge_weights: np.ndarray | None = None

    def in_degrees(self) -> np.ndarray:
        return np.diff(self.t_row_offsets.astype(np.int64))

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
    """Upload (once per host graph object and device) and return the device CSR."""
    if isinstance(g, DeviceGraph):
        return g
    import torch
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    try:
        per = _cache.get(g)
    except TypeError:
        per = None
    dg = per.get(str(dev)) if per is not None else None
    if dg is None:
        dg = DeviceGraph.from_host(g, dev)
        try:
            _cache.setdefault(g, {})[str(dev)] = dg
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


# ------------------------------------------------------------ construction --
def _stable_group(keys_dev, num_keys, torch):
    """(indptr int64[num_keys+1], perm int32[n]) of a stable counting sort."""
    from . import _lib
    n = int(keys_dev.numel())
    dev = keys_dev.device
    indptr = torch.empty(num_keys + 1, dtype=torch.int64, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    wsb = _lib.lib().fgl_stable_group_ws_bytes(num_keys)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("fgl_stable_group", keys_dev.data_ptr(), n, num_keys, indptr.data_ptr(), perm.data_ptr(), None,
              ws.data_ptr(), wsb, st)
    return indptr, perm[:n]


def _gather(perm, a=None, b=None, torch=None):
    from . import _lib
    n = int(perm.numel())
    ao = torch.empty(max(n, 1), dtype=torch.int32, device=perm.device) if a is not None else None
    bo = torch.empty(max(n, 1), dtype=torch.float32, device=perm.device) if b is not None else None
    _lib.call("fgl_gather_i32_f32", perm.data_ptr(), n, a.data_ptr() if a is not None else None,
              b.data_ptr() if b is not None else None, ao.data_ptr() if ao is not None else None,
              bo.data_ptr() if bo is not None else None, torch.cuda.current_stream().cuda_stream)
    return (ao[:n] if ao is not None else None), (bo[:n] if bo is not None else None)


def device_from_edges(num_nodes: int, src, dst, weights=None, device="cuda"):
    """CSR + transpose of an edge list on the GPU.  Canonical order is
    lexicographic (src, dst), stable for duplicate edges (graph.py:163-171):
    an LSD pass of two stable counting sorts (by dst, then by src) gives it;
    the transpose is a stable counting sort of that list by dst.  Returns
    device tensors (row_offsets, cols, w, t_row_offsets, t_cols, t_w)."""
    import torch
    n = int(num_nodes)
    s = torch.as_tensor(np.ascontiguousarray(src).astype(np.int32)).to(device)
    d = torch.as_tensor(np.ascontiguousarray(dst).astype(np.int32)).to(device)
    w = None if weights is None else torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float32)).to(device)
    _, p1 = _stable_group(d, n, torch)                    # grouped by dst
    s1, _ = _gather(p1, s, None, torch)
    row_offsets, p2 = _stable_group(s1, n, torch)         # then by src (stable): (src, dst) order
    order, _ = _gather(p2, p1, None, torch)
    cols, wf = _gather(order, d, w, torch)
    srcs, _ = _gather(order, s, None, torch)
    t_row_offsets, pt = _stable_group(cols, n, torch)     # transpose: by dst, then src
    t_cols, t_w = _gather(pt, srcs, wf, torch)
    return row_offsets, cols, wf, t_row_offsets, t_cols, t_w


def from_edges(num_nodes: int, src, dst, weights=None) -> Graph:
    """Drop-in for graph.from_edges (graph.py:151-183): duplicates and self
    loops kept, canonical (src, dst) order; built on the GPU, returned with
    the reference's host dtypes (uint64 offsets / columns, f32 weights)."""
    src = np.asarray(src, dtype=np.uint64)
    dst = np.asarray(dst, dtype=np.uint64)
    if src.shape != dst.shape:
        raise ValidationError("src/dst length mismatch")
    if weights is not None:
        weights = np.asarray(weights, dtype=np.float32)
        if weights.shape != src.shape:
            raise ValidationError("weights length mismatch")
    if src.size and max(int(src.max()), int(dst.max())) >= num_nodes:
        raise ValidationError("edge endpoint out of range")
    if num_nodes >= 2**31 or src.size >= 2**31:
        raise ValidationError("device CSR build needs num_nodes and num_edges below 2^31")
    ro, c, w, tro, tc, tw = device_from_edges(num_nodes, src, dst, weights)
    h = lambda t, dt: t.cpu().numpy().astype(dt)
    return Graph(num_nodes=int(num_nodes), num_edges=int(src.size), row_offsets=h(ro, np.uint64),
                 col_indices=h(c, np.uint64), edge_weights=None if w is None else h(w, np.float32),
                 t_row_offsets=h(tro, np.uint64), t_col_indices=h(tc, np.uint64),
                 t_edge_weights=None if tw is None else h(tw, np.float32))


# ------------------------------------------------------------- MGL1 files --
MAGIC = b"MGL1"
_U64 = np.dtype("<u8")
_F32 = np.dtype("<f4")


def save_binary(g, path) -> None:
    """Serialize a graph in the reference's MGL1 layout (graph.py:293-307):
    magic, u64 [num_nodes, num_edges], flag bytes (weights, transpose), then
    row_offsets, col_indices, [weights], t_row_offsets, t_col_indices, [t_weights]."""
    has_w = getattr(g, "edge_weights", None) is not None
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(np.array([g.num_nodes, g.num_edges], dtype=_U64).tobytes())
        fh.write(bytes([1 if has_w else 0, 1]))
        fh.write(np.ascontiguousarray(g.row_offsets, dtype=_U64).tobytes())
        fh.write(np.ascontiguousarray(g.col_indices, dtype=_U64).tobytes())
        if has_w:
            fh.write(np.ascontiguousarray(g.edge_weights, dtype=_F32).tobytes())
        fh.write(np.ascontiguousarray(g.t_row_offsets, dtype=_U64).tobytes())
        fh.write(np.ascontiguousarray(g.t_col_indices, dtype=_U64).tobytes())
        if has_w:
            fh.write(np.ascontiguousarray(g.t_edge_weights, dtype=_F32).tobytes())


def _read_array(fh, count, dtype):
    nbytes = count * dtype.itemsize
    buf = fh.read(nbytes)
    if len(buf) != nbytes:
        raise FormatError(f"truncated file: wanted {nbytes} bytes, got {len(buf)}")
    return np.frombuffer(buf, dtype=dtype).copy()


def load_binary(path) -> Graph:
    """Inverse of save_binary (graph.py:318-351), bit-exact round trip; a file
    without the transpose has it rebuilt by the GPU CSR build."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MAGIC:
            raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
        header = _read_array(fh, 2, _U64)
        num_nodes, num_edges = int(header[0]), int(header[1])
        flags = fh.read(2)
        if len(flags) != 2:
            raise FormatError("truncated file: missing flag bytes")
        has_w, has_t = flags[0] != 0, flags[1] != 0
        row_offsets = _read_array(fh, num_nodes + 1, _U64)
        col_indices = _read_array(fh, num_edges, _U64)
        weights = _read_array(fh, num_edges, _F32) if has_w else None
        if has_t:
            t_row_offsets = _read_array(fh, num_nodes + 1, _U64)
            t_col_indices = _read_array(fh, num_edges, _U64)
            t_weights = _read_array(fh, num_edges, _F32) if has_w else None
            return Graph(num_nodes=num_nodes, num_edges=num_edges, row_offsets=row_offsets,
                         col_indices=col_indices, edge_weights=weights, t_row_offsets=t_row_offsets,
                         t_col_indices=t_col_indices, t_edge_weights=t_weights)
    src = np.repeat(np.arange(num_nodes, dtype=np.uint64), np.diff(row_offsets.astype(np.int64)))
    return from_edges(num_nodes, src, col_indices, weights)
