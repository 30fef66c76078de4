"""Mini-batch GNN training on B200: drop-in for ``minigl.trainer``.

The epoch driver keeps the reference's structure (trainer.py:246-349): a
fixed Philox partition of the training IDs into batches, windows of
``window_n`` batches, per-batch sampling seed ``derive_seed(seed, 13, j)``,
Match-Reorder of each window, then forward / fp64 loss / backward / SGD per
batch in schedule order.  Everything per batch runs in HBM through
``libfastgl_b200.so``:

  sample  fgl_sample_window     whole window in one launch sequence
  map     (fused into sampling) window rows + frontier indices
  io      fgl_match_counts + greedy order, fgl_gather_rows (Match delta load)
  prepare fgl_prepare_layer     block CSR + stable transpose + GCN weights
  compute fgl_spmm / fgl_dense_fwd / fgl_softmax_xent / fgl_dense_bwd / fgl_sgd

GCN runs on the sampled *block* graph: model layer i (hop h = H-1-i) computes
only the rows of hop h's frontier -- every other row of the reference's
all-rows layer (trainer.py:182-195) is a zero aggregation whose value no later
layer or loss term reads.  GIN needs every row (its self term carries rows
forward), so it runs the full unique-node layout like the reference.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ValidationError
from .graph import device_graph
from .memsim import BatchTraffic, CostParams, TrafficReport, t_memory_aware, t_naive
from .sampler import Fanouts, WindowSampler, counts_layout, derive_seed, make_epoch_batches
from .store import HostFeatureStore

__all__ = ["ModelConfig", "PipelineFlags", "EpochStats", "TrainReport", "train", "derive_seed",
           "init_params", "DeviceModel", "Pipeline", "StaticFeatureCache", "phase_breakdown", "PHASES"]

PHASES = ("sample", "map", "io_sim", "compute")


def _ld(d: int) -> int:
    return (int(d) + 3) // 4 * 4


class _NeedAlloc(RuntimeError):
    """A work buffer must grow while a CUDA graph is being captured."""


@dataclass
class ModelConfig:
    """Architecture and schedule knobs (trainer.py:45-79)."""

    layer_dims: tuple
    fanouts: Fanouts
    arch: str = "gcn"
    batch_size: int = 64
    window_n: int = 8
    epochs: int = 20
    lr: float = 0.3
    seed: int = 0
    map_workers: int = 1
    tiles: object = None

    def __post_init__(self):
        if not isinstance(self.fanouts, Fanouts):
            self.fanouts = Fanouts(self.fanouts)
        self.layer_dims = tuple(int(d) for d in self.layer_dims)
        if self.arch not in ("gcn", "gin", "sage"):
            raise ValidationError(f"unknown arch {self.arch!r}")
        if len(self.layer_dims) < 2 or any(d < 1 for d in self.layer_dims):
            raise ValidationError("layer_dims needs input dim, optional hiddens, and classes")
        if len(self.fanouts) != len(self.layer_dims) - 1:
            raise ValidationError(
                f"{len(self.fanouts)} fanouts for {len(self.layer_dims) - 1} aggregation layers")
        if self.batch_size < 1 or self.window_n < 1 or self.epochs < 1:
            raise ValidationError("batch_size, window_n and epochs must be >= 1")
        if self.lr < 0:
            raise ValidationError("lr must be non-negative")

    @property
    def num_layers(self) -> int:
        return len(self.layer_dims) - 1


@dataclass
class PipelineFlags:
    """IO-path switches (trainer.py:82-89); only ``reorder`` changes the trajectory."""

    match: bool = True
    reorder: bool = True
    memory_aware: bool = True


@dataclass
class EpochStats:
    loss: float
    accuracy: float
    traffic: TrafficReport
    phase_seconds: dict
    modeled_fetch_seconds: float = 0.0


@dataclass
class TrainReport:
    config: ModelConfig
    flags: PipelineFlags
    epochs: list = field(default_factory=list)

    @property
    def losses(self) -> list:
        return [e.loss for e in self.epochs]


def init_params(layer_dims, seed: int):
    """Glorot-normal weights, zero biases from Philox(derive_seed(seed, 101))
    (trainer.py:145-153).  Host-side, once per run."""
    rng = np.random.Generator(np.random.Philox(derive_seed(seed, 101)))
    params = []
    for d_in, d_out in zip(layer_dims, layer_dims[1:]):
        scale = np.sqrt(2.0 / (d_in + d_out))
        w = (rng.standard_normal((d_in, d_out)) * scale).astype(np.float32)
        params.append([w, np.zeros(d_out, dtype=np.float32)])
    return params


class DeviceModel:
    """All weights/biases in one flat f32 buffer (one allreduce bucket for DP),
    with a matching flat gradient buffer."""

    def __init__(self, layer_dims, params, device="cuda"):
        import torch
        self.dims = tuple(layer_dims)
        sizes = []
        for a, b in zip(self.dims, self.dims[1:]):
            sizes += [a * b, b]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        flat = np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in params])
        self.flat = torch.from_numpy(flat.astype(np.float32)).to(device)
        self.grad = torch.zeros_like(self.flat)

    def _ptr(self, t, k):
        return t.data_ptr() + 4 * int(self.offsets[k])

    def W(self, i):
        return self._ptr(self.flat, 2 * i)

    def b(self, i):
        return self._ptr(self.flat, 2 * i + 1)

    def dW(self, i):
        return self._ptr(self.grad, 2 * i)

    def db(self, i):
        return self._ptr(self.grad, 2 * i + 1)

    def to_numpy(self):
        f = self.flat.cpu().numpy()
        out = []
        for i, (a, b) in enumerate(zip(self.dims, self.dims[1:])):
            o = self.offsets[2 * i]
            out.append([f[o : o + a * b].reshape(a, b).copy(), f[o + a * b : o + a * b + b].copy()])
        return out

    def grads_numpy(self):
        g = self.grad.cpu().numpy()
        out = []
        for i, (a, b) in enumerate(zip(self.dims, self.dims[1:])):
            o = self.offsets[2 * i]
            out.append([g[o : o + a * b].reshape(a, b).copy(), g[o + a * b : o + a * b + b].copy()])
        return out


def _feature_array(feats):
    """The [N, d] array of a FeatureMatrix (graph.py:90-114), ndarray or tensor."""
    if hasattr(feats, "dim") and hasattr(feats, "num_nodes") and not callable(feats.dim):
        return feats.data
    return feats


def greedy_order(m: np.ndarray) -> list:
    """Greedy chain of schedule.py:92-113 on a match-degree matrix: batch 0
    first, then the unused batch with the highest degree to the last one;
    ties and non-positive rows resolve to the lowest index."""
    n = len(m)
    order, used, cur = [0], np.zeros(n, dtype=bool), 0
    used[0] = True
    for _ in range(n - 1):
        row = np.where(used, -1.0, m[cur])
        h = int(np.argmax(row))
        if row[h] <= 0.0:
            h = int(np.flatnonzero(~used)[0])
        order.append(h)
        used[h] = True
        cur = h
    return order


class StaticFeatureCache:
    """Static-degree feature cache in HBM (memsim.py:110-126 made real): the
    floor(ratio * N) highest-degree nodes (ties: lower node id) keep their
    feature rows in an HBM table; ``slot[g]`` is the row of node g in that
    table or -1.  The loader (fgl_gather_rows_cached) serves a row that Match
    does not cover from the table instead of the host link, and counts the
    hits (bytes_served_by_cache of simulate_epoch_io, memsim.py:129-186)."""

    POLICIES = ("none", "static-degree")

    def __init__(self, dg, host_feats: int, d, ld, cache_ratio: float, policy: str = "static-degree",
                 device="cuda"):
        import torch
        if not 0.0 <= cache_ratio <= 1.0:
            raise ValidationError("cache_ratio must be within [0, 1]")
        if policy not in self.POLICIES:
            raise ValidationError(f"unknown cache policy {policy!r}")
        n = int(dg.num_nodes)
        self.k = int(np.floor(cache_ratio * n)) if policy == "static-degree" else 0
        self.ratio, self.policy, self.ld = cache_ratio, policy, ld
        self.slot = torch.full((n,), -1, dtype=torch.int32, device=device)
        self.table = torch.zeros((max(self.k, 1), ld), dtype=torch.float32, device=device)
        if self.k > 0:
            off = dg.row_offsets
            deg = (off[1:] - off[:-1]).to(torch.int64)
            # stable sort on -degree: equal degrees keep ascending node id
            top = torch.argsort(-deg, stable=True)[: self.k].to(torch.int32).contiguous()
            self.slot[top.long()] = torch.arange(self.k, dtype=torch.int32, device=device)
            self.nodes = top
            _lib.call("fgl_gather_rows", host_feats, ld, d, top.data_ptr(), self.k, None, None, 0,
                      None, ld, self.table.data_ptr(), ld, None, torch.cuda.current_stream().cuda_stream)
        else:
            self.nodes = torch.zeros(0, dtype=torch.int32, device=device)

    def mask_numpy(self, n):
        m = np.zeros(n, dtype=bool)
        m[self.nodes.cpu().numpy()] = True
        return m


class Pipeline:
    """Device-resident training pipeline for one graph / feature store / model.

    ``feature_store``: "device" keeps the feature matrix in HBM; "host" keeps
    it in pinned host memory and every x0 row not reused through Match crosses
    the host link (zero-copy reads, config 4 of BASELINE.json).
    """

    MAX_MATCH_WINDOW = 16

    def __init__(self, g, feats, labels, cfg: ModelConfig, flags: PipelineFlags | None = None,
                 device="cuda", feature_store="device", params=None, dist=None, direct_x0=None,
                 cache_ratio: float = 0.0, cache_policy: str = "static-degree", dense_ctas: int = 74):
        import torch
        self.torch = torch
        self.cfg = cfg
        # SM budget of the tensor-core dense kernels while run_windows keeps
        # three other streams busy (fgl_set_dense_ctas; 0 = every SM)
        self.dense_ctas = int(os.environ.get("FGL_DENSE_CTAS", dense_ctas))
        self.flags = flags or PipelineFlags()
        # device-side limits of a window (checked before any allocation): the
        # match-degree pass keeps all pair counts of a window in registers
        # (<= 16 batches), the depth-major relayout of GIN / SAGE ranks up to
        # 64 batches per pass
        if self.flags.reorder and cfg.window_n > self.MAX_MATCH_WINDOW:
            raise ValidationError(f"window_n {cfg.window_n} > {self.MAX_MATCH_WINDOW}: the GPU match-degree "
                                  f"schedule handles at most {self.MAX_MATCH_WINDOW} batches per window")
        if cfg.arch != "gcn" and cfg.window_n > 64:
            raise ValidationError(f"window_n {cfg.window_n} > 64 is not supported for arch {cfg.arch!r}")
        self.device = device
        self.dist = dist
        self.dg = device_graph(g, device)
        if isinstance(feats, HostFeatureStore):
            # a pinned (possibly node-shared) host table: the loader reads it zero-copy
            self.store = feats
            feature_store = "host"
            self.d0 = feats.dim
        else:
            data = _feature_array(feats)
            ft = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data, np.float32))
            self.d0 = int(ft.shape[1])
            self.store = HostFeatureStore.private(ft) if feature_store == "host" else None
        if self.d0 != cfg.layer_dims[0]:
            raise ValidationError(f"feature dim {self.d0} != model input dim {cfg.layer_dims[0]}")
        self.ldf = _ld(self.d0)
        self.feature_store = feature_store
        if self.store is not None:
            self.feats = self.store.table
            self.feats_ptr = self.store.dev_ptr
        else:
            dev = torch.zeros((ft.shape[0], self.ldf), dtype=torch.float32, device=device)
            dev[:, : self.d0].copy_(ft.to(device) if not ft.is_cuda else ft)
            self.feats = dev
            self.feats_ptr = dev.data_ptr()
        lab = labels if isinstance(labels, torch.Tensor) else torch.from_numpy(np.asarray(labels, dtype=np.int64))
        self.labels = lab.to(device=device, dtype=torch.int64)
        self.sampler = WindowSampler(self.dg, cfg.fanouts, cfg.batch_size, cfg.window_n, device=device,
                                     window_rows=cfg.arch != "gcn", depth_layout=cfg.arch != "gcn")
        out = _lib.i64_array([0, 0, 0])
        _lib.call("fgl_sample_ws_bitmaps", self.dg.num_nodes, cfg.window_n, self.sampler.fcap,
                  self.sampler.uniq_cap, out)
        self.bm_off, self.prefix_off, self.words = int(out[0]), int(out[1]), int(out[2])
        self.model = DeviceModel(cfg.layer_dims, params if params is not None else init_params(cfg.layer_dims, cfg.seed), device)
        self.L = cfg.num_layers
        self.H = len(cfg.fanouts)
        # row-length bound of model layer 0 (rows of the last hop hold <= its fanout edges)
        self._max_fan = min(16, int(cfg.fanouts.counts[-1]))
        self.compact = cfg.arch == "gcn"
        # direct_x0: with the feature table resident in HBM, the layer-0
        # aggregation gathers neighbour rows straight from the table (the x0
        # staging copy -- and with it the Match reuse, which only saves host-
        # link traffic -- is skipped).  Host-resident features always go
        # through the Match delta loader.
        if direct_x0 is None:
            direct_x0 = False
        self.direct_x0 = bool(direct_x0) and feature_store == "device" and self.compact
        # GIN / SAGE (depth-major rows): the layer-0 aggregation and its root
        # term read the table through the batch's row -> node id map
        # (fgl_spmm_ids) instead of a gathered x0 block (FGL_DIRECT_IDS=0: x0)
        d4 = (cfg.layer_dims[0] + 3) // 4
        self.direct_ids = (bool(direct_x0) and feature_store == "device" and not self.compact and 8 < d4 <= 32
                           and os.environ.get("FGL_DIRECT_IDS", "1") != "0")
        self.pairs = torch.zeros(120, dtype=torch.int64, device=device)
        # rows read from the feature store / served by the static cache, per
        # schedule position of the window (BatchTraffic rows of memsim.py:52-60)
        self.loaded = torch.zeros(max(cfg.window_n, 1), dtype=torch.int64, device=device)
        self.cache_hits = torch.zeros(max(cfg.window_n, 1), dtype=torch.int64, device=device)
        self.cache = None
        if cache_ratio > 0.0 or cache_policy not in StaticFeatureCache.POLICIES:
            if feature_store != "host":
                raise ValidationError("the static feature cache fronts a host-resident feature store")
            self.cache = StaticFeatureCache(self.dg, self.feats_ptr, self.d0, self.ldf, cache_ratio, cache_policy,
                                            device)
        self.loss_dev = torch.zeros(max(cfg.window_n, 1), dtype=torch.float64, device=device)
        dims = cfg.layer_dims
        # one weight-gradient workspace per layer: the upper layers' weight
        # gradients run on a side stream concurrently with the backward chain
        self.bwd_ws_l = [torch.empty(_lib.lib().fgl_dense_bwd_ws_bytes(a, b), dtype=torch.uint8, device=device)
                         for a, b in zip(dims, dims[1:])]
        self.bwd_ws = self.bwd_ws_l[0]
        self._wg_stream = None
        self._cs = None  # stream being issued on inside run_windows
        self._capturing = False
        self.graph_fallbacks = 0
        self._fuse_top = os.environ.get("FGL_FUSE_TOP", "1") != "0"
        self._keep_l0_transpose = False  # tests that inspect layer 0's transpose set this
        self.xent_ws = torch.empty(_lib.lib().fgl_softmax_xent_ws_bytes(), dtype=torch.uint8, device=device)
        self._bufs = {}
        self._graveyard = []
        self.gpu_launches = 0
        self._pre_h0 = None
        self._pre_h0_win = None
        self._agg_stream = None
        self._execs = {}
        if self._world() > 1 and hasattr(self.dist, "warmup"):
            self.dist.warmup(device)

    # ------------------------------------------------------------ buffers --
    def _buf(self, name, rows, cols, dtype=None):
        torch = self.torch
        dtype = dtype or torch.float32
        need = max(int(rows), 1) * int(cols)
        t = self._bufs.get(name)
        if t is None or t.numel() < need or t.dtype != dtype:
            if self._capturing:
                raise _NeedAlloc(name)  # no allocation inside a graph capture: run this batch eagerly
            if t is not None:
                # buffers are used from two streams: a replaced one may still be
                # read by queued kernels, so it is kept alive, never recycled
                self._graveyard.append(t)
            t = torch.empty(int(need * 1.25) + 64, dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t

    @property
    def stream(self):
        cs = self._cs
        return cs.cuda_stream if cs is not None else self.torch.cuda.current_stream().cuda_stream

    def _cur(self):
        """The stream work is being issued on (cached inside run_windows: a
        torch.cuda.current_stream() call costs ~10 us of host time)."""
        cs = self._cs
        return cs if cs is not None else self.torch.cuda.current_stream()

    def _call(self, name, *args):
        _lib.call(name, *args)
        self.gpu_launches += 1

    # ----------------------------------------------------------- schedule --
    def schedule(self, win, nb: int) -> list:
        """Match-degree matrix on the GPU from the batches' node bitmaps, greedy
        chain on the host (schedule.py:68-113)."""
        if not self.flags.reorder or nb < 2:
            return list(range(nb))
        pre = getattr(win, "pairs_host", None)
        if pre is not None:  # read back behind the sampler (_sample_async)
            with _host_trace()("wait pairs"):
                pre[1].synchronize()
            pairs = pre[0].numpy().copy()
        else:
            ws = win.s.ws.data_ptr()
            self._call("fgl_match_counts", ws + self.bm_off, self.words, nb, self.pairs.data_ptr(), self.stream)
            pairs = self.pairs.cpu().numpy()
        sizes = [win.unique_range(b)[1] - win.unique_range(b)[0] for b in range(nb)]
        m = np.zeros((nb, nb), dtype=np.float64)
        for i in range(nb):
            for j in range(i + 1, nb):
                k = i * 16 - i * (i + 1) // 2 + (j - i - 1)
                m[i, j] = m[j, i] = int(pairs[k]) / min(sizes[i], sizes[j])
        self.last_match = m
        return greedy_order(m)

    # ------------------------------------------------------------ prepare --
    def prepare(self, win, slot: int = 0) -> list:
        """Block CSR (+ stable transpose, GCN weights) of every model layer for
        the whole window (trainer.py:165-179).  `slot` selects one of two
        buffer sets, so the next window can be prepared while this one trains."""
        torch = self.torch
        s = self.sampler
        layers = [None] * self.L
        for h in range(self.H):
            e0, e1 = win.hop_edges(h)
            nnz = e1 - e0
            if self.compact:
                lt, ls = s.tgt_front, s.src_front
                rows = win.front_total(h)
                cols = win.front_total(h + 1) if h + 1 < self.H else win.unique_total()
            else:
                lt, ls = s.tgt_row, s.src_row
                rows = cols = win.unique_total()
            grouped = (not self.compact) and s.depth_layout
            rows, cols = max(rows, 1), max(cols, 1)
            # model layer 0 (hop H-1, the largest) needs no transpose: nothing
            # aggregates a gradient back into the input features
            need_t = h != self.H - 1 or self._keep_l0_transpose
            lay = {
                "indptr": self._buf(f"ip{h}s{slot}", rows + 1, 1, torch.int64),
                "w": self._buf(f"w{h}s{slot}", max(nnz, 1), 1),
                "t_indptr": self._buf(f"tip{h}s{slot}", cols + 1, 1, torch.int64) if need_t else None,
                "t_col": self._buf(f"tc{h}s{slot}", max(nnz, 1), 1, torch.int32) if need_t else None,
                "t_w": self._buf(f"tw{h}s{slot}", max(nnz, 1), 1) if need_t else None,
                "col": ls.data_ptr() + 4 * e0,
                "col_global": s.src.data_ptr() + 4 * e0,
                "nnz": nnz,
            }
            tptr = (lambda k: lay[k].data_ptr() if lay[k] is not None else None)
            arch_code = {"gin": 0, "gcn": 1, "sage": 2}[self.cfg.arch]
            if grouped:  # depth-major targets are grouped but not ascending
                colb = self._buf(f"colg{h}s{slot}", max(nnz, 1), 1, torch.int32)
                lay["col"] = colb.data_ptr()
                wsb = _lib.lib().fgl_prepare_layer_grouped_ws_bytes(nnz, rows, cols)
                pws = self._buf(f"pws{h}s{slot}", wsb, 1, torch.uint8)
                self._call("fgl_prepare_layer_grouped", lt.data_ptr() + 4 * e0, ls.data_ptr() + 4 * e0, nnz, rows,
                           cols, arch_code, lay["indptr"].data_ptr(), colb.data_ptr(), lay["w"].data_ptr(),
                           tptr("t_indptr"), tptr("t_col"), tptr("t_w"), pws.data_ptr(), wsb, self.stream)
            else:
                wsb = _lib.lib().fgl_prepare_layer_ws_bytes(nnz, rows, cols)
                pws = self._buf(f"pws{h}s{slot}", wsb, 1, torch.uint8)
                self._call("fgl_prepare_layer", lt.data_ptr() + 4 * e0, ls.data_ptr() + 4 * e0, nnz, rows,
                           cols, arch_code, lay["indptr"].data_ptr(),
                           lay["w"].data_ptr(), tptr("t_indptr"), tptr("t_col"),
                           tptr("t_w"), pws.data_ptr(), wsb, self.stream)
            layers[self.H - 1 - h] = lay
        return layers

    # ---------------------------------------------------------- row spaces --
    def _rows(self, win, i, b):
        """(first, last) row of batch b in model layer i's output row space."""
        if self.compact:
            return win.front_range(self.H - 1 - i, b)
        u0, u1 = win.unique_range(b)
        if win.s.depth_layout:  # depth-major rows: layer i needs a prefix
            return u0, u0 + win.prefix_rows(i, b)
        return u0, u1

    def _in_base(self, win, i, b):
        """Row of batch b's first input row in layer i's input index space."""
        if i == 0 or not self.compact:
            return win.unique_range(b)[0]
        return win.front_range(self.H - i, b)[0]

    # -------------------------------------------------------------- batch --
    def _world(self) -> int:
        return int(getattr(self.dist, "world", 1)) if self.dist is not None else 1

    def _graphs_on(self) -> bool:
        """CUDA graphs unless disabled, or a collective that cannot be
        captured (gloo) sits inside the chain."""
        return (os.environ.get("FGL_GRAPH", "1") != "0"
                and (self._world() <= 1 or bool(getattr(self.dist, "capturable", False))))

    def _graph_mode(self) -> bool:
        return self._cs is not None and self._graphs_on()

    def _graphed(self, stream, slot: int, fn):
        """Run fn() -- work issued on `stream` only, no host reads of device
        data, no cross-stream events leaving it -- as one CUDA graph through
        executable-graph slot `slot`; eager fallback if the capture fails."""
        import os
        if not self._graphs_on() or str(slot) not in os.environ.get("FGL_GRAPH_SLOTS", "0,1,2,3").split(","):
            return fn()
        st = stream.cuda_stream
        _lib.call("fgl_capture_begin", st)
        self._capturing = True
        try:
            r = fn()
        except Exception:  # noqa: BLE001 - discard the capture, run eagerly
            self._capturing = False
            _lib.lib().fgl_capture_abort(st)
            self.graph_fallbacks += 1
            return fn()
        self._capturing = False
        try:
            _lib.call("fgl_capture_end_launch", self._exec(slot), st)
        except Exception:  # noqa: BLE001 - instantiate / launch refused: run eagerly
            self.graph_fallbacks += 1
            return fn()
        return r

    def _exec(self, slot: int):
        """This pipeline's executable graph for sequence `slot` (0 batch chain,
        1 prepare, 2 sampler, 3 window chain), created on first use."""
        h = self._execs.get(slot)
        if h is None:
            import ctypes
            p = ctypes.c_void_p()
            _lib.call("fgl_exec_create", ctypes.byref(p))
            h = self._execs[slot] = p.value
        return h

    def __del__(self):
        execs = getattr(self, "_execs", None) or {}
        try:
            lib = _lib.lib()
            for h in execs.values():
                lib.fgl_exec_destroy(h)
            for h in (getattr(self, "_xevs", None) or {}).values():
                lib.fgl_event_destroy(h)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass
        self._execs = {}
        self._xevs = {}

    def batch_step(self, win, b, prev, slot, layers, x0_slot):
        """Load x0, forward, loss, backward, SGD for batch b of the window.

        Inside run_windows the batch's chain is captured and replayed as one
        CUDA graph (fgl_capture_*): the same kernels with the same arguments,
        fewer host calls and shorter launch gaps.  A capture that fails (a
        buffer has to grow, an unexpected path) is aborted and the batch runs
        eagerly."""
        if not self._graph_mode():
            return self._batch_step_body(win, b, prev, slot, layers, x0_slot)
        cur = self._cs
        # dependencies on other streams are taken before the capture starts
        pre = (self._pre_h0.get(b) if (self._pre_h0 is not None and self._pre_h0_win is win) else None)
        if pre is not None and pre[1] is not None:
            cur.wait_event(pre[1])
        st = cur.cuda_stream
        _lib.call("fgl_capture_begin", st)
        self._capturing = True
        try:
            self._batch_step_body(win, b, prev, slot, layers, x0_slot, external_done=True)
        except Exception:  # noqa: BLE001 - any failure: discard the capture, run eagerly
            self._capturing = False
            _lib.lib().fgl_capture_abort(st)
            self.graph_fallbacks += 1
            return self._batch_step_body(win, b, prev, slot, layers, x0_slot, external_done=True)
        self._capturing = False
        try:
            _lib.call("fgl_capture_end_launch", self._exec(0), st)
        except Exception:  # noqa: BLE001 - instantiate / launch refused: run eagerly
            self.graph_fallbacks += 1
            self._batch_step_body(win, b, prev, slot, layers, x0_slot, external_done=True)

    def _gather_x0(self, win, b, prev, slot, x0_slot):
        """x0 = feats[unique_nodes of batch b] (trainer.py:315) in the batch's
        row order: rows the previous batch (`prev`, Match) already holds are
        copied from its block, the rest come from the static HBM cache or the
        feature store (loader.cu); per-position row counts go to
        loaded / cache_hits.  With direct_x0 the layer-0 aggregation reads the
        HBM table itself and there is no x0 block."""
        s = self.sampler
        st = self.stream
        if self.direct_x0 or self.direct_ids:
            return self.feats
        u0, u1 = win.unique_range(b)
        U = u1 - u0
        ws = s.ws.data_ptr()
        x0 = self._buf(f"x0_{x0_slot}", U, self.ldf)
        if prev is not None:
            p0 = win.unique_range(prev)[0]
            prev_bm = ws + self.bm_off + 4 * prev * self.words
            prev_pf = ws + self.prefix_off + 4 * prev * self.words
            prev_x = self._bufs[f"x0_{1 - x0_slot}"].data_ptr()
        else:
            p0, prev_bm, prev_pf, prev_x = 0, None, None, None
        row_map = s.row_map.data_ptr() if (prev_bm is not None and s.depth_layout) else None
        cached = self.cache is not None and self.cache.k > 0
        self._call("fgl_gather_rows_cached", self.feats_ptr, self.ldf, self.d0,
                   s.unique.data_ptr() + 4 * u0, U, prev_bm, prev_pf, p0, prev_x, self.ldf, row_map,
                   self.cache.slot.data_ptr() if cached else None, self.cache.table.data_ptr() if cached else None,
                   self.ldf, x0.data_ptr(), self.ldf, self.loaded.data_ptr() + 8 * slot,
                   self.cache_hits.data_ptr() + 8 * slot if cached else None, st)
        return x0

    def _batch_step_body(self, win, b, prev, slot, layers, x0_slot, external_done=False):
        torch = self.torch
        s = self.sampler
        m = self.model
        dims = self.cfg.layer_dims
        st = self.stream
        x0 = self._gather_x0(win, b, prev, slot, x0_slot)
        # forward
        s0, s1 = int(win.seed_off_host[b]), int(win.seed_off_host[b + 1])
        # the top layer in one kernel (GCN: with its aggregation; GIN / SAGE: the
        # aggregation with its root term stays in fgl_spmm, the kernel reads H)
        top_fused = (self.L >= 2 and dims[-2] <= 64 and dims[-1] <= 192
                     and self._fuse_top
                     and (self._rows(win, self.L - 1, b)[1] - self._rows(win, self.L - 1, b)[0]) == s1 - s0)
        X, ldx = x0, self.ldf
        H_bufs, Y_bufs, ns = [], [], []
        for i in range(self.L):
            din, dout = dims[i], dims[i + 1]
            r0, r1 = self._rows(win, i, b)
            n = r1 - r0
            lay = layers[i]
            pre = (self._pre_h0.get(b) if (i == 0 and self._pre_h0 is not None and self._pre_h0_win is win)
                   else None)
            if pre is not None:
                # layer-0 aggregation was run ahead on the aggregation stream
                Hb, ev = pre
                if not external_done and ev is not None:
                    self._cur().wait_event(ev)
            elif i == self.L - 1 and top_fused and self.compact:
                # the fused top-layer kernel gathers H = A X itself
                Hb = None
                top_agg = (lay["indptr"].data_ptr() + 8 * r0, lay["col"], lay["w"].data_ptr(),
                           self._in_base(win, i, b), X.data_ptr(), ldx)
            else:
                Hb = self._buf(f"h{i}", n, _ld(din))
                self_x = X.data_ptr() if not self.compact else None
                col, base = lay["col"], self._in_base(win, i, b)
                if i == 0 and self.direct_x0:
                    col, base = lay["col_global"], 0
                if i == 0 and self.direct_ids:
                    # batch-local row c -> node id unique[u0 + c]: neighbour rows
                    # and the root term straight from the HBM table
                    u0 = win.unique_range(b)[0]
                    self._call("fgl_spmm_ids", lay["indptr"].data_ptr() + 8 * r0, lay["col"], lay["w"].data_ptr(),
                               n, base, self.feats_ptr, self.ldf, s.unique.data_ptr() + 4 * u0, r0 - u0, 1,
                               Hb.data_ptr(), _ld(din), din, st)
                else:
                    self._call("fgl_spmm", lay["indptr"].data_ptr() + 8 * r0, col, lay["w"].data_ptr(), n,
                               base, X.data_ptr(), ldx, self_x, ldx, Hb.data_ptr(), _ld(din), din, st)
                if i == self.L - 1 and top_fused:
                    top_agg = (None, None, None, 0, Hb.data_ptr(), _ld(din))
            if i == self.L - 1 and top_fused:
                Yb = None  # the fused top-layer kernel computes the logits itself
            else:
                Yb = self._buf(f"y{i}", n, _ld(dout))
                self._call("fgl_dense_fwd", Hb.data_ptr(), _ld(din), n, din, m.W(i), m.b(i), dout,
                           Yb.data_ptr(), _ld(dout), 1 if i < self.L - 1 else 0, st)
            H_bufs.append(Hb)
            Y_bufs.append(Yb)
            ns.append(n)
            X, ldx = Yb, _ld(dout)
        s0, s1 = int(win.seed_off_host[b]), int(win.seed_off_host[b + 1])
        C = dims[-1]
        r0, _ = self._rows(win, self.L - 1, b)
        rows_ptr = (s.seed_front if self.compact else s.seed_rows).data_ptr() + 4 * s0
        wg_done = []
        side = self._side_wgrad_stream()
        first_bwd = self.L - 1
        if top_fused:
            # top layer: logits, loss, dH and the weight-gradient partials in
            # one launch; the partial reduction runs on the side stream
            it = self.L - 1
            din = dims[it]
            dHt = self._buf(f"dh{it}", ns[it], _ld(din))
            B = s1 - s0
            wsb = _lib.lib().fgl_top_layer_ws_bytes(B, din, C)
            tws = self._buf(f"top_ws{slot % 2}", wsb, 1, torch.uint8)
            red = side.cuda_stream if side is not None else None
            a_ip, a_col, a_w, a_base, a_x, a_ld = top_agg
            self._call("fgl_top_layer", a_x, a_ld, rows_ptr, r0,
                       s.seeds_dev.data_ptr() + 4 * s0, self.labels.data_ptr(), B, din, C, m.W(it), m.b(it),
                       dHt.data_ptr(), _ld(din), m.dW(it), m.db(it), self.loss_dev.data_ptr() + 8 * slot,
                       tws.data_ptr(), wsb, a_ip, a_col, a_w, a_base, st, red)
            if side is not None:
                ready = torch.cuda.Event()
                ready.record(self._cur())
                side.wait_event(ready)
                self._call("fgl_top_layer_reduce", B, din, C, m.dW(it), m.db(it),
                           self.loss_dev.data_ptr() + 8 * slot, tws.data_ptr(), side.cuda_stream)
                done = torch.cuda.Event()
                done.record(side)
                wg_done.append(done)
        else:
            # loss over the seed rows of the last layer
            dY = self._buf("dy_last", ns[-1], _ld(C))
            if not self.compact:
                self._call("fgl_fill_rows", dY.data_ptr(), _ld(C), ns[-1], C, None, 0, st)
            self._call("fgl_softmax_xent", Y_bufs[-1].data_ptr(), _ld(C), rows_ptr, r0,
                       s.seeds_dev.data_ptr() + 4 * s0, self.labels.data_ptr(), s1 - s0, C,
                       dY.data_ptr(), _ld(C), self.loss_dev.data_ptr() + 8 * slot,
                       self.xent_ws.data_ptr(), self.xent_ws.numel(), st)
        # backward.  Layer i > 0: its weight gradient (dW, db) only feeds the
        # SGD step, so it runs on a side stream while the chain continues with
        # dH = dZ W^T -> transposed aggregation -> layer i-1; the SGD waits for
        # all of them.  Same kernels and inputs: results are unchanged.
        dX, lddx = (None, 0) if top_fused else (dY, _ld(C))
        for i in range(first_bwd, -1, -1):
            din, dout = dims[i], dims[i + 1]
            n = ns[i]
            mask = Y_bufs[i].data_ptr() if i < self.L - 1 else None
            dH = self._buf(f"dh{i}", n, _ld(din)) if i > 0 else None
            ws_i = self.bwd_ws_l[i]
            if top_fused and i == self.L - 1:
                pass  # dH / dW / db of the top layer came from fgl_top_layer
            elif i > 0 and side is not None:
                ready = torch.cuda.Event()
                ready.record(self._cur())
                side.wait_event(ready)
                self._call("fgl_dense_bwd", H_bufs[i].data_ptr(), _ld(din), n, din, m.W(i), dout,
                           dX.data_ptr(), lddx, mask, _ld(dout), m.dW(i), m.db(i), None, _ld(din),
                           ws_i.data_ptr(), ws_i.numel(), side.cuda_stream)
                done = torch.cuda.Event()
                done.record(side)
                wg_done.append(done)
                self._call("fgl_dense_dgrad", dX.data_ptr(), lddx, mask, _ld(dout), n, m.W(i), din, dout,
                           dH.data_ptr(), _ld(din), st)
            else:
                self._call("fgl_dense_bwd", H_bufs[i].data_ptr(), _ld(din), n, din, m.W(i), dout,
                           dX.data_ptr(), lddx, mask, _ld(dout), m.dW(i), m.db(i),
                           dH.data_ptr() if dH is not None else None, _ld(din), ws_i.data_ptr(),
                           ws_i.numel(), st)
            if i > 0:
                lay = layers[i]
                q0, q1 = self._rows(win, i - 1, b)
                nx = q1 - q0
                dXn = self._buf(f"dx{i}", nx, _ld(din))
                col_base = self._rows(win, i, b)[0]
                prefix = (not self.compact) and s.depth_layout
                self_x = dH.data_ptr() if (not self.compact and not prefix) else None
                self._call("fgl_spmm", lay["t_indptr"].data_ptr() + 8 * q0, lay["t_col"].data_ptr(),
                           lay["t_w"].data_ptr(), nx, col_base, dH.data_ptr(), _ld(din), self_x,
                           _ld(din), dXn.data_ptr(), _ld(din), din, st)
                if prefix:  # root term dx += dh on the layer's own (prefix) rows only
                    self._call("fgl_add_rows", dXn.data_ptr(), _ld(din), dH.data_ptr(), _ld(din), n, din, st)
                dX, lddx = dXn, _ld(din)
        cur = self._cur()
        for ev in wg_done:
            cur.wait_event(ev)
        world = self._world()
        if world > 1:
            # synchronous DP: the SUM of the ranks' gradients, the 1/W of the
            # mean folded into the step size (one collective per batch)
            self.dist.allreduce_sum(self.model.grad)
        self._call("fgl_sgd", m.flat.data_ptr(), m.grad.data_ptr(), m.grad.numel(), float(self.cfg.lr) / world, st)

    def _side_wgrad_stream(self):
        import os
        if os.environ.get("FGL_SIDE_WGRAD", "1") == "0":
            return None
        if self._wg_stream is None:
            torch = self.torch
            try:
                lo, hi = torch.cuda.Stream.priority_range()
                self._wg_stream = torch.cuda.Stream(device=self.device, priority=min(lo, hi))
            except Exception:  # noqa: BLE001 - no priority support
                self._wg_stream = torch.cuda.Stream(device=self.device)
        return self._wg_stream

    # --------------------------------------------- layer-0 run-ahead --
    def _xev_on(self) -> bool:
        """Per-batch cross-graph events between the prepare graph and the
        window's chain graph (FGL_XEV=0: the chain waits for the whole prepare)."""
        return (self._graphs_on() and os.environ.get("FGL_GRAPH_WINDOW", "1") != "0"
                and os.environ.get("FGL_XEV", "1") != "0")

    def _xev(self, slot: int, key):
        """External-flag CUDA event (slot, key): key "csr" = the window's block
        CSRs done, j = the j-th layer-0 aggregation of the window done."""
        if not hasattr(self, "_xevs"):
            self._xevs = {}
        h = self._xevs.get((slot, key))
        if h is None:
            import ctypes
            p = ctypes.c_void_p()
            _lib.call("fgl_event_create", ctypes.byref(p))
            h = self._xevs[(slot, key)] = p.value
        return h

    def _launch_l0_aggs(self, win, order, layers, slot: int = 0, stream=None):
        """Layer 0's aggregation H0 = A_0 X (features straight from the HBM
        table) depends on the sampled window only, not on the weights, so
        the aggregations of ALL batches of the window are issued up front on a
        separate stream; each batch step waits for its own event.  The wide
        random-gather SpMMs then overlap the latency-bound dense / backward
        kernels of earlier batches.  Results are identical (same kernel, same
        inputs).  Only for the direct-x0 compact layout (features in HBM)."""
        torch = self.torch
        if not ((self.direct_x0 and self.compact) or self.direct_ids):
            self._pre_h0 = None
            return
        if stream is None:
            if self._agg_stream is None:
                self._agg_stream = torch.cuda.Stream(device=self.device)
            stream = self._agg_stream
            ready = torch.cuda.Event()
            ready.record()  # prepare of this window (and every earlier batch step) is ordered before
            stream.wait_event(ready)
        lay = layers[0]
        din = self.cfg.layer_dims[0]
        pre = {}
        xev = self._xev_on()
        with torch.cuda.stream(stream):
            st = stream.cuda_stream
            if xev:  # the window's block CSRs are complete here
                _lib.call("fgl_event_record_ext", self._xev(slot, "csr"), st)
            for j, b in enumerate(order):
                r0, r1 = self._rows(win, 0, b)
                n = r1 - r0
                Hb = self._buf(f"h0_run{j}s{slot}", n, _ld(din))
                if self.direct_ids:  # GIN / SAGE: table rows through the row -> node id map, root term included
                    u0 = win.unique_range(b)[0]
                    self._call("fgl_spmm_ids", lay["indptr"].data_ptr() + 8 * r0, lay["col"], lay["w"].data_ptr(), n,
                               self._in_base(win, 0, b), self.feats_ptr, self.ldf, win.s.unique.data_ptr() + 4 * u0,
                               r0 - u0, 1, Hb.data_ptr(), _ld(din), din, st)
                elif self.ldf <= 128:
                    # rows hold <= fanout edges: the software-pipelined short-row
                    # kernel (bit-identical to fgl_spmm)
                    self._call("fgl_spmm_gather", lay["indptr"].data_ptr() + 8 * r0, lay["col_global"],
                               lay["w"].data_ptr(), n, 0, self.feats_ptr, self.ldf, int(self.feats.shape[0]),
                               Hb.data_ptr(), _ld(din), din, self._max_fan, st)
                else:
                    self._call("fgl_spmm", lay["indptr"].data_ptr() + 8 * r0, lay["col_global"], lay["w"].data_ptr(),
                               n, 0, self.feats_ptr, self.ldf, None, self.ldf, Hb.data_ptr(), _ld(din), din,
                               st)
                if xev:  # batch j's H0 is complete here (an event-record node inside the prepare graph)
                    _lib.call("fgl_event_record_ext", self._xev(slot, j), st)
                if self._capturing:  # graph-captured: `prepped` or the per-batch external events order it
                    pre[b] = (Hb, None)
                else:
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    pre[b] = (Hb, ev)
        self._pre_h0 = pre
        self._pre_h0_win = win

    def row_length_histograms(self, win, order, layers) -> np.ndarray:
        """[position, layer, row length] counts of every executed batch's
        model-layer CSR rows (the input of trainer.py:230-242's fetch model);
        rows without edges land in bin 0.  One device->host read."""
        torch = self.torch
        nb, nbin = len(order), max(int(f) for f in self.cfg.fanouts) + 1
        out = torch.zeros((nb, self.L, nbin), dtype=torch.int64, device=self.device)
        for j, b in enumerate(order):
            for i in range(self.L):
                r0, r1 = self._rows(win, i, b)
                if r1 <= r0:
                    continue
                ip = layers[i]["indptr"][r0 : r1 + 1]
                out[j, i] = torch.bincount((ip[1:] - ip[:-1]).clamp_(max=nbin - 1), minlength=nbin)[:nbin]
        return out.cpu().numpy()

    # ------------------------------------------------------------- window --
    def run_window(self, seed_lists, rng_seeds, phase=None):
        """Sample, schedule, prepare and train one window; returns (order,
        per-batch device losses tensor view)."""
        torch = self.torch
        tick = (lambda: (torch.cuda.synchronize(), time.perf_counter())[1]) if phase is not None else None
        t0 = tick() if tick else 0.0
        win = self.sampler.sample(seed_lists, rng_seeds)
        self.gpu_launches += 1
        win.host_counts()
        nb = len(seed_lists)
        t1 = tick() if tick else 0.0
        order = self.schedule(win, nb)
        t2 = tick() if tick else 0.0
        layers = self.prepare(win)
        self._launch_l0_aggs(win, order, layers)
        t3 = tick() if tick else 0.0
        for j, b in enumerate(order):
            prev = order[j - 1] if (j > 0 and self.flags.match) else None
            self.batch_step(win, b, prev, j, layers, j % 2)
        if tick:
            t4 = tick()
            phase["sample"] += t1 - t0
            phase["io_sim"] += t2 - t1
            phase["map"] += t3 - t2
            phase["compute"] += t4 - t3
        self.last_window = win
        self.last_layers = layers
        return order, self.loss_dev[:nb]

    # --------------------------------------------------------- pipelined --
    # windows sampled ahead of the one being trained (>= 1: window w is
    # always sampled before it is popped)
    LOOKAHEAD = max(1, int(os.environ.get("FGL_LOOKAHEAD", "2")))

    def _sample_async(self, seed_lists, rng_seeds, slot):
        """Stage + launch the window sampler of slot `slot` (LOOKAHEAD + 1
        samplers in rotation) on the sampling stream (asynchronous)."""
        torch = self.torch
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(device=self.device)
            self._samplers = [self.sampler] + [
                WindowSampler(self.dg, self.cfg.fanouts, self.cfg.batch_size, self.cfg.window_n, device=self.device,
                              window_rows=self.cfg.arch != "gcn", depth_layout=self.cfg.arch != "gcn")
                for _ in range(self.LOOKAHEAD)]
        smp = self._samplers[slot]
        done = getattr(self, "_slot_done", {}).get(slot)
        if done is not None:  # the compute of the window that last used this slot
            self._side.wait_event(done)
        with torch.cuda.stream(self._side):
            nb, off = smp.stage(seed_lists, rng_seeds)
            win = self._graphed(self._side, 2, lambda: smp.run(nb, off, stream=self._side))
            win.sampled = torch.cuda.Event()
            win.sampled.record(self._side)
            # the window's counts and match matrix, read back right behind the
            # sampler: when the window comes up for training (LOOKAHEAD windows
            # later) its schedule needs no device round trip, so the prepare
            # and chain launches are not held behind a busy GPU
            if not hasattr(self, "_pin_counts"):
                self._pin_counts = [torch.zeros(self._counts_cap(), dtype=torch.int64).pin_memory()
                                    for _ in range(self.LOOKAHEAD + 1)]
                self._pairs_dev = [torch.zeros_like(self.pairs) for _ in range(self.LOOKAHEAD + 1)]
                self._pin_pairs = [torch.zeros(self.pairs.numel(), dtype=torch.int64).pin_memory()
                                   for _ in range(self.LOOKAHEAD + 1)]
            win.prefetch_counts(self._pin_counts[slot], self._side)
            if self.flags.reorder and nb >= 2:
                self._call("fgl_match_counts", smp.ws.data_ptr() + self.bm_off, self.words, nb,
                           self._pairs_dev[slot].data_ptr(), self._side.cuda_stream)
                self._pin_pairs[slot].copy_(self._pairs_dev[slot], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self._side)
                win.pairs_host = (self._pin_pairs[slot], ev)
        self.gpu_launches += 1
        return win

    def _counts_cap(self) -> int:
        H, nb = self.H, self.cfg.window_n
        return counts_layout(H, nb)["len"] + nb * (H + 1)

    def run_windows(self, windows):
        """Train a sequence of windows [(seed_lists, rng_seeds), ...] on three
        streams: sampling runs LOOKAHEAD windows ahead, the block CSRs and
        layer-0 aggregations of window w run on a prepare stream under window
        w-1's compute, and the weight-dependent chain runs on a high-priority
        stream.  Yields (order, device losses) per window; numerically
        identical to run_window applied in sequence (the dense kernels' SM
        budget only changes their grid)."""
        torch = self.torch
        windows = list(windows)
        if not windows:
            return
        caller = torch.cuda.current_stream()
        _lib.call("fgl_set_dense_ctas", self.dense_ctas)
        try:
            yield from self._run_windows(windows, caller)
        finally:
            _lib.call("fgl_set_dense_ctas", 0)

    def _run_windows(self, windows, caller):
        import collections
        torch = self.torch
        # the weight-dependent chain (dense / backward / SGD, many short
        # kernels) is the critical path: it runs on a HIGH-priority stream so
        # its CTAs are scheduled ahead of the wide sampling / aggregation
        # kernels of the side streams whenever SMs free up
        if not hasattr(self, "_main"):
            try:
                lo, hi = torch.cuda.Stream.priority_range()
            except Exception:  # noqa: BLE001 - no priority support: default priority
                lo = hi = 0
            self._main = torch.cuda.Stream(device=self.device, priority=min(lo, hi))
            self._prep = torch.cuda.Stream(device=self.device)
            self._io = torch.cuda.Stream(device=self.device)
            self._prep_done = {}
        if not hasattr(self, "_slot_done"):
            self._slot_done = {}
        self._main.wait_stream(caller)
        nsmp = self.LOOKAHEAD + 1
        trace = _host_trace()
        pending = collections.deque()
        for k in range(min(self.LOOKAHEAD, len(windows))):
            pending.append(self._sample_async(*windows[k], slot=k % nsmp))

        def issue_prepare(w):
            """Schedule window w (its counts and match matrix were read back
            behind its sampler) and queue its block CSRs and layer-0
            aggregations on the prepare stream.  Issued right after window
            w-1's chain, so the prepare runs under that whole chain."""
            with trace(f"window {w}: counts + schedule"):
                win = pending.popleft()
                nb = win.num_batches
                self.sampler = win.s
                self._io.wait_event(win.sampled)
                with torch.cuda.stream(self._io):
                    self._cs = self._io
                    win.host_counts()
                    order = self.schedule(win, nb)
                    self._cs = None
            with trace(f"window {w}: prepare issue"):
                slot = w % 2
                self._prep.wait_event(win.sampled)
                if slot in self._prep_done:  # prepare buffers of this slot: window w-2 has trained
                    self._prep.wait_event(self._prep_done[slot])
                with torch.cuda.stream(self._prep):
                    self._cs = self._prep

                    def _prep_work():
                        lay = self.prepare(win, slot)
                        self._launch_l0_aggs(win, order, lay, slot, stream=self._prep)
                        return lay
                    layers = self._graphed(self._prep, 1, _prep_work)
                    prepped = torch.cuda.Event()
                    prepped.record(self._prep)
                    self._cs = None
            return win, order, layers, prepped, self._pre_h0

        nxt = issue_prepare(0)
        for w in range(len(windows)):
            win, order, layers, prepped, pre_h0 = nxt
            nb = win.num_batches
            self.sampler = win.s
            self._pre_h0, self._pre_h0_win = pre_h0, win
            # the caller may still be reading the previous window's losses
            # (e.g. an asynchronous copy of the yielded view): order this
            # window's writes after everything the caller has queued
            self._main.wait_stream(caller)
            with trace(f"window {w}: chain issue"):
                with torch.cuda.stream(self._main):
                    self._cs = self._main
                    pslot = w % 2
                    xev = self._xev_on() and self._pre_h0 is not None and self._pre_h0_win is win
                    if not xev:
                        self._main.wait_event(prepped)
                    if self._graph_mode() and os.environ.get("FGL_GRAPH_WINDOW", "1") != "0":
                        # the whole window's chain (8 batch steps) as ONE graph:
                        # no launch gaps between batches either
                        for b in order:
                            pre = self._pre_h0.get(b) if (self._pre_h0 is not None and self._pre_h0_win is win) else None
                            if pre is not None and pre[1] is not None:
                                self._main.wait_event(pre[1])

                        def _window_chain():
                            st = self._main.cuda_stream
                            if xev:  # event-wait nodes on the prepare graph: batch j starts once its H0 is ready
                                _lib.call("fgl_stream_wait_ext", st, self._xev(pslot, "csr"))
                            for j, b in enumerate(order):
                                if xev:
                                    _lib.call("fgl_stream_wait_ext", st, self._xev(pslot, j))
                                prev = order[j - 1] if (j > 0 and self.flags.match) else None
                                self._batch_step_body(win, b, prev, j, layers, j % 2, external_done=True)
                        self._graphed(self._main, 3, _window_chain)
                    else:
                        for j, b in enumerate(order):
                            prev = order[j - 1] if (j > 0 and self.flags.match) else None
                            self.batch_step(win, b, prev, j, layers, j % 2)
                    ev = torch.cuda.Event()
                    ev.record(self._main)
                self._cs = None
            self._slot_done[w % nsmp] = ev
            self._prep_done[w % 2] = ev
            self.last_window = win
            # next: the sampler LOOKAHEAD windows ahead (its slot was freed by
            # window w-1's chain), then window w+1's prepare -- both queued
            # while this window's chain runs on the device
            with trace(f"window {w}: sampler issue"):
                if w + self.LOOKAHEAD < len(windows):
                    k = w + self.LOOKAHEAD
                    pending.append(self._sample_async(*windows[k], slot=k % nsmp))
            if w + 1 < len(windows):
                nxt = issue_prepare(w + 1)
                self.sampler = win.s
                self._pre_h0, self._pre_h0_win = pre_h0, win
            caller.wait_stream(self._main)  # the caller's stream sees this window's losses / weights
            yield order, self.loss_dev[:nb]
        self.sampler = self._samplers[0]


def _host_trace():
    """Host-side ranges for tools/timeline.py (FGL_HOST_TRACE=1: profiler
    record_function annotations; otherwise no-op context managers)."""
    mode = os.environ.get("FGL_HOST_TRACE", "0")
    if mode == "1":
        import torch
        return torch.profiler.record_function
    import contextlib
    if mode == "2":  # perf_counter sums per phase in HOST_TIMES (tools/host_phases.py)
        @contextlib.contextmanager
        def timed(name):
            t = time.perf_counter()
            yield
            key = name.split(": ", 1)[-1]
            HOST_TIMES[key] = HOST_TIMES.get(key, 0.0) + time.perf_counter() - t
        return timed
    return lambda name: contextlib.nullcontext()


HOST_TIMES: dict = {}


def train(g, feats, labels, cfg: ModelConfig, flags: PipelineFlags | None = None, *,
          train_ids=None, val_ids=None, cost_params=None, feature_store="device",
          cache_ratio: float = 0.0, cache_policy: str = "static-degree") -> TrainReport:
    """Drop-in for trainer.train (trainer.py:246-349): same batch stream, same
    schedule, per-batch SGD; loss/accuracy per epoch; IO accounting from the
    loader's real row counts."""
    import torch
    flags = flags or PipelineFlags()
    labels_np = np.asarray(labels, dtype=np.int64)
    n = int(g.num_nodes)
    if len(labels_np) != n:
        raise ValidationError("labels length must equal num_nodes")
    fdata = _feature_array(feats)
    if fdata.shape[0] != n:
        raise ValidationError("feature rows must equal num_nodes")
    if fdata.shape[1] != cfg.layer_dims[0]:
        raise ValidationError(f"feature dim {fdata.shape[1]} != model input dim {cfg.layer_dims[0]}")
    if labels_np.max() >= cfg.layer_dims[-1]:
        raise ValidationError("label exceeds the class count")
    if train_ids is None or val_ids is None:
        rng = np.random.Generator(np.random.Philox(derive_seed(cfg.seed, 7)))
        perm = rng.permutation(n).astype(np.uint64)
        cut = max(1, int(0.8 * n))
        train_ids = perm[:cut] if train_ids is None else np.asarray(train_ids, np.uint64)
        val_ids = perm[cut:] if val_ids is None else np.asarray(val_ids, np.uint64)
    train_ids = np.asarray(train_ids, dtype=np.uint64)
    val_ids = np.asarray(val_ids, dtype=np.uint64)
    if train_ids.size == 0:
        raise ValidationError("training split is empty")
    if cache_ratio > 0.0:
        feature_store = "host"  # the cache fronts the host-resident store (memsim.py:129-186)
    pipe = Pipeline(g, feats, labels_np, cfg, flags, feature_store=feature_store, cache_ratio=cache_ratio,
                    cache_policy=cache_policy)
    seed_batches = make_epoch_batches(g, train_ids, cfg.batch_size, derive_seed(cfg.seed, 11))
    windows = [seed_batches[i : i + cfg.window_n] for i in range(0, len(seed_batches), cfg.window_n)]
    report = TrainReport(config=cfg, flags=flags)
    d = pipe.d0
    params = cost_params or CostParams()
    params.validate()
    fetch = t_memory_aware if flags.memory_aware else t_naive
    node_bytes = 4 * d
    for _ in range(cfg.epochs):
        phase = dict.fromkeys(PHASES, 0.0)
        loss_sum, seen, base = 0.0, 0, 0
        per_batch, modeled = [], 0.0
        for win_seeds in windows:
            rs = [derive_seed(cfg.seed, 13, base + j) for j in range(len(win_seeds))]
            base += len(win_seeds)
            pipe.loaded.zero_()
            pipe.cache_hits.zero_()
            order, losses = pipe.run_window([w.astype(np.int64) for w in win_seeds], rs, phase)
            lv = losses.cpu().numpy()
            loaded = pipe.loaded.cpu().numpy()
            hits = pipe.cache_hits.cpu().numpy()
            win = pipe.last_window
            hist = pipe.row_length_histograms(win, order, pipe.last_layers)
            for j, bi in enumerate(order):
                loss_sum += float(lv[j])  # sum of per-seed losses = mean * batch size
                seen += len(win_seeds[bi])
                u0, u1 = win.unique_range(bi)
                ld, hit = int(loaded[j]), int(hits[j])
                per_batch.append(BatchTraffic(position=len(per_batch), loaded_nodes=ld, bytes_h2d=ld * node_bytes,
                                              bytes_cache=hit * node_bytes,
                                              bytes_match=(u1 - u0 - ld - hit) * node_bytes))
                # trainer.py:230-242 per batch: layers in order, row lengths ascending
                total = 0.0
                for i in range(pipe.L):
                    for f in np.flatnonzero(hist[j, i]):
                        if f > 0:
                            total += int(hist[j, i, f]) * fetch(int(f), cfg.layer_dims[i], params)
                modeled += total
        traffic = TrafficReport.from_batches(per_batch, params)
        acc = evaluate(pipe, g, val_ids) if val_ids.size else float("nan")
        report.epochs.append(EpochStats(loss=loss_sum / max(seen, 1), accuracy=acc, traffic=traffic,
                                        phase_seconds=phase, modeled_fetch_seconds=modeled))
    report.pipeline = pipe
    return report


def evaluate(pipe: Pipeline, g, eval_ids) -> float:
    """Sampled-neighbourhood accuracy with fixed draws derive_seed(seed,17,i)
    (trainer.py:352-365): forward only, argmax over the seed rows."""
    import torch
    cfg = pipe.cfg
    correct = total = 0
    eval_ids = np.asarray(eval_ids, dtype=np.uint64)
    ev = getattr(pipe, "_eval_sampler", None)
    if ev is None:
        ev = WindowSampler(pipe.dg, cfg.fanouts, cfg.batch_size, 1, device=pipe.device)
        pipe._eval_sampler = ev
    saved = pipe.sampler
    pipe.sampler = ev
    try:
        for i in range(0, len(eval_ids), cfg.batch_size):
            seeds = eval_ids[i : i + cfg.batch_size]
            win = ev.sample([seeds.astype(np.int64)], [derive_seed(cfg.seed, 17, i)])
            win.host_counts()
            layers = pipe.prepare(win)
            logits, rows = pipe.forward_only(win, 0, layers)
            pred = logits[rows].argmax(dim=1)
            lab = pipe.labels[torch.from_numpy(seeds.astype(np.int64)).to(pipe.device)]
            correct += int((pred == lab).sum().item())
            total += len(seeds)
    finally:
        pipe.sampler = saved
    return correct / max(total, 1)


def _forward_only(self, win, b, layers):
    """Forward pass of batch b; returns (logits tensor [n, C], seed row index tensor)."""
    torch = self.torch
    s = self.sampler
    m = self.model
    dims = self.cfg.layer_dims
    st = self.stream
    u0, u1 = win.unique_range(b)
    x0 = self._buf("x0_eval", u1 - u0, self.ldf)
    self._call("fgl_gather_rows", self.feats_ptr, self.ldf, self.d0, s.unique.data_ptr() + 4 * u0,
               u1 - u0, None, None, 0, None, self.ldf, x0.data_ptr(), self.ldf, None, st)
    X, ldx = x0, self.ldf
    for i in range(self.L):
        din, dout = dims[i], dims[i + 1]
        r0, r1 = self._rows(win, i, b)
        n = r1 - r0
        Hb = self._buf(f"h{i}", n, _ld(din))
        self._call("fgl_spmm", layers[i]["indptr"].data_ptr() + 8 * r0, layers[i]["col"],
                   layers[i]["w"].data_ptr(), n, self._in_base(win, i, b), X.data_ptr(), ldx,
                   X.data_ptr() if not self.compact else None, ldx, Hb.data_ptr(), _ld(din), din, st)
        Yb = self._buf(f"ye{i}", n, _ld(dout))
        self._call("fgl_dense_fwd", Hb.data_ptr(), _ld(din), n, din, m.W(i), m.b(i), dout, Yb.data_ptr(),
                   _ld(dout), 1 if i < self.L - 1 else 0, st)
        X, ldx = Yb, _ld(dout)
    C = dims[-1]
    n_last = self._rows(win, self.L - 1, b)
    n = n_last[1] - n_last[0]
    logits = X[: n * _ld(C)].view(n, _ld(C))[:, :C]
    s0, s1 = int(win.seed_off_host[b]), int(win.seed_off_host[b + 1])
    rows = (s.seed_front if self.compact else s.seed_rows)[s0:s1].long() - n_last[0]
    return logits, rows


Pipeline.forward_only = _forward_only


def phase_breakdown(report: TrainReport) -> dict:
    """Percentage of wall time per pipeline phase (trainer.py:368-376)."""
    if not report.epochs:
        raise ValidationError("cannot break down an empty report")
    totals = {p: sum(e.phase_seconds[p] for e in report.epochs) for p in PHASES}
    overall = sum(totals.values())
    if overall <= 0:
        raise ValidationError("report has no recorded time")
    return {p: 100.0 * t / overall for p, t in totals.items()}
