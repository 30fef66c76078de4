"""k-hop sampler: drop-in for ``minigl.sampler`` backed by the Fused-Map CUDA
window sampler (csrc/sampler.cu via fgl_sample_window).

``sample_khop(g, seeds, fanouts, seed)`` keeps the reference signature and
returns the reference's ``SubgraphBatch`` layout (uint64 global IDs, f32
weights), bit-exact with sampler.py:120-139.  :class:`WindowSampler` is the
device-level API the trainer uses: a whole window of batches per call, all
results left in HBM (int32 IDs) with per-batch offsets.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ValidationError
from .graph import device_graph

__all__ = ["Fanouts", "SubgraphBatch", "sample_khop", "sample_random_walk", "make_epoch_batches",
           "philox_key", "derive_seed", "WindowSampler", "DeviceWindow", "WalkSampler"]


def derive_seed(base: int, *parts: int) -> int:
    """Child seed (trainer.py:40-42): first word of SeedSequence((base, *parts))."""
    return int(np.random.SeedSequence((base, *parts)).generate_state(1)[0])


def philox_key(seed: int) -> tuple[int, int]:
    """Key of np.random.Philox(seed) = SeedSequence(seed).generate_state(2)."""
    k = np.random.SeedSequence(int(seed)).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


@dataclass
class Fanouts:
    """Per-hop neighbor sample counts; ``counts[0]`` expands the seeds (sampler.py:27-44)."""

    counts: tuple[int, ...]

    def __init__(self, counts):
        object.__setattr__(self, "counts", tuple(int(c) for c in counts))
        if not self.counts:
            raise ValidationError("fanouts must not be empty")
        if any(c < 1 for c in self.counts):
            raise ValidationError("every fanout must be >= 1")

    def __len__(self):
        return len(self.counts)

    def __iter__(self):
        return iter(self.counts)


@dataclass
class SubgraphBatch:
    """Sampled mini-batch, field-compatible with sampler.py:47-68."""

    seeds: np.ndarray
    layers: list
    unique_nodes: np.ndarray
    local_layers: list = field(default_factory=list)
    num_local: int = 0

    @property
    def num_unique(self) -> int:
        return len(self.unique_nodes)

    def num_sampled_edges(self) -> int:
        return sum(len(t) for t, _, _ in self.layers)


def _validate_seeds(num_nodes: int, seeds) -> np.ndarray:
    seeds = np.asarray(seeds, dtype=np.uint64)
    if seeds.size == 0:
        raise ValidationError("seeds must not be empty")
    if seeds.max() >= np.uint64(num_nodes):
        raise ValidationError("seed id out of range")
    return seeds


def counts_layout(H: int, nb: int) -> dict:
    """Offsets of the FGL_CNT_* sections (include/fastgl_b200.h)."""
    fo = H * nb + 1
    uo = fo + H * (nb + 1)
    do = uo + nb + 1
    so = do + nb
    return {"front": fo, "uniq": uo, "draws": do, "status": so, "len": so + 1}


@dataclass
class DeviceWindow:
    """Results of one sampled window, resident in HBM.

    Edge arrays are hop-major / batch-minor; ``tgt_row``/``src_row`` are window
    rows (batch b's local ID + its unique offset), ``tgt_front``/``src_front``
    index hop h's / hop h+1's frontier list (last hop: window row)."""

    num_batches: int
    num_hops: int
    s: "WindowSampler"
    seed_off_host: np.ndarray
    _host_counts: np.ndarray | None = None

    _pinned = None  # (pinned host copy of the counts, event) queued by prefetch_counts

    def _counts_len(self) -> int:
        n = counts_layout(self.num_hops, self.num_batches)["len"]
        if self.s.depth_layout:
            n += self.num_batches * (self.num_hops + 1)
        return n

    def prefetch_counts(self, pinned, stream) -> None:
        """Queue the counts read-back on `stream` right behind the sampler
        (asynchronous, into the pinned buffer `pinned`): host_counts then only
        waits for an event that completed long before the window trains."""
        import torch
        n = self._counts_len()
        pinned[:n].copy_(self.s.counts[:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        self._pinned = (pinned, ev)

    def host_counts(self) -> np.ndarray:
        """One device->host read of the counts vector (the window's only sync);
        with the depth layout the per-(batch, depth) counts follow it."""
        if self._host_counts is None:
            n = self._counts_len()
            if self._pinned is not None:
                pinned, ev = self._pinned
                from .trainer import _host_trace
                with _host_trace()("wait counts"):
                    ev.synchronize()
                c = pinned[:n].numpy().copy()
            else:
                c = self.s.counts[:n].cpu().numpy()
            _lib.status_error(int(c[counts_layout(self.num_hops, self.num_batches)["status"]]),
                              "fgl_sample_window")
            self._host_counts = c
        return self._host_counts

    def edge_range(self, hop: int, b: int):
        c = self.host_counts()
        k = hop * self.num_batches + b
        return int(c[k]), int(c[k + 1])

    def hop_edges(self, hop: int):
        c = self.host_counts()
        return int(c[hop * self.num_batches]), int(c[(hop + 1) * self.num_batches])

    def front_range(self, hop: int, b: int):
        c = self.host_counts()
        k = counts_layout(self.num_hops, self.num_batches)["front"] + hop * (self.num_batches + 1) + b
        return int(c[k]), int(c[k + 1])

    def front_total(self, hop: int) -> int:
        return self.front_range(hop, self.num_batches - 1)[1]

    def unique_range(self, b: int):
        c = self.host_counts()
        u0 = counts_layout(self.num_hops, self.num_batches)["uniq"]
        return int(c[u0 + b]), int(c[u0 + b + 1])

    def unique_total(self) -> int:
        return self.unique_range(self.num_batches - 1)[1]

    def draws(self, b: int) -> int:
        c = self.host_counts()
        return int(c[counts_layout(self.num_hops, self.num_batches)["draws"] + b])

    def total_edges(self) -> int:
        return int(self.host_counts()[self.num_hops * self.num_batches])

    def prefix_rows(self, layer: int, b: int) -> int:
        """Depth layout: rows of model layer `layer` for batch b = nodes of
        depth <= H-1-layer (a prefix of the batch's block)."""
        c = self.host_counts()
        o = counts_layout(self.num_hops, self.num_batches)["len"] + b * (self.num_hops + 1)
        return int(c[o : o + self.num_hops - layer].sum())

    def hop_draws(self, hop: int) -> int:
        """Philox draws (= candidates = sum of frontier degrees) of one hop;
        measurement helper, computed on the device."""
        f = self.frontier(hop).long()
        off = self.s.g.row_offsets
        return int((off[f + 1] - off[f]).sum().item())

    def frontier(self, hop: int):
        return self.s.frontier[hop * self.s.fcap : hop * self.s.fcap + self.front_total(hop)]

    def to_batch(self, b: int) -> SubgraphBatch:
        """Host SubgraphBatch of batch b in the reference's dtypes."""
        s = self.s
        layers, local = [], []
        u0, u1 = self.unique_range(b)
        for h in range(self.num_hops):
            e0, e1 = self.edge_range(h, b)
            t = s.tgt[e0:e1].cpu().numpy().astype(np.uint64)
            src = s.src[e0:e1].cpu().numpy().astype(np.uint64)
            w = s.wgt[e0:e1].cpu().numpy()
            layers.append((t, src, w))
            if s.tgt_row is not None:
                local.append((s.tgt_row[e0:e1].cpu().numpy().astype(np.int64) - u0,
                              s.src_row[e0:e1].cpu().numpy().astype(np.int64) - u0, w))
        s0, s1 = int(self.seed_off_host[b]), int(self.seed_off_host[b + 1])
        uniq = s.unique[u0:u1].cpu().numpy().astype(np.uint64)
        seeds = s.seeds_dev[s0:s1].cpu().numpy().astype(np.uint64)
        return SubgraphBatch(seeds=seeds, layers=layers, unique_nodes=uniq, local_layers=local,
                             num_local=len(uniq) if local else 0)


class WindowSampler:
    """Device sampler for windows of up to ``max_batches`` batches of up to
    ``max_batch_size`` seeds.  Buffers are allocated once (worst-case bounds
    from fgl_sample_bounds) and reused; results of a call stay valid until the
    next call."""

    def __init__(self, dgraph, fanouts, max_batch_size: int, max_batches: int = 1,
                 local_ids: bool = True, device="cuda", window_rows: bool = True, depth_layout: bool = False):
        import torch
        self.torch = torch
        self.g = dgraph
        self.fanouts = Fanouts(fanouts)
        self.H = len(self.fanouts)
        self.max_nb = int(max_batches)
        self.max_bs = int(max_batch_size)
        self.device = device
        out = (ctypes.c_int64 * 5)()
        sizes = _lib.i64_array([self.max_bs] * self.max_nb)
        _lib.call("fgl_sample_bounds", self.g.num_nodes, sizes, self.max_nb,
                  _lib.i32_array(self.fanouts.counts), self.H, out)
        self.edge_cap, self.fcap, self.uniq_cap, self.ws_bytes, self.counts_len = (int(x) for x in out)
        e = self.edge_cap
        i32 = dict(dtype=torch.int32, device=device)
        opt = (lambda n: torch.empty(n, **i32)) if local_ids else (lambda n: None)
        self.tgt = torch.empty(e, **i32)
        self.src = torch.empty(e, **i32)
        self.wgt = torch.empty(e, dtype=torch.float32, device=device)
        # window rows (unique-rank IDs) are only needed by the all-rows layout
        # (GIN / SAGE) and the drop-in API; the compact GCN layout uses the
        # frontier indices alone, and skipping the rows saves a rank lookup per edge
        optr = opt if window_rows else (lambda n: None)
        self.tgt_row, self.src_row = optr(e), optr(e)
        self.tgt_front, self.src_front = opt(e), opt(e)
        self.unique = torch.empty(self.uniq_cap, **i32)
        self.frontier = torch.empty(self.H * self.fcap, **i32)
        nseed = self.max_nb * self.max_bs
        self.seed_rows, self.seed_front = optr(nseed), opt(nseed)
        self.ws = torch.zeros(self.ws_bytes, dtype=torch.uint8, device=device)
        self.seeds_dev = torch.empty(nseed, **i32)
        self.seed_off = torch.empty(self.max_nb + 1, dtype=torch.int64, device=device)
        self.keys = torch.empty(2 * self.max_nb, dtype=torch.int64, device=device)
        # counts vector + per-(batch, depth) counts of the depth layout right after it
        self.counts = torch.empty(self.counts_len + self.max_nb * (self.H + 1), dtype=torch.int64, device=device)
        self.depth_layout = bool(depth_layout and window_rows and local_ids)
        self.row_map = None
        if self.depth_layout:
            self.row_map = torch.empty(max(self.uniq_cap, 1), dtype=torch.int32, device=device)
            rb = _lib.lib().fgl_depth_relayout_ws_bytes(self.uniq_cap)
            self.relayout_ws = torch.empty(rb, dtype=torch.uint8, device=device)
            out3 = _lib.i64_array([0, 0, 0])
            _lib.call("fgl_sample_ws_bitmaps", dgraph.num_nodes, self.max_nb, self.fcap, self.uniq_cap, out3)
            self._bm_all_off, self._prefix_off, self._words = int(out3[0]), int(out3[1]), int(out3[2])
        # pinned staging of a window's inputs (seeds | offsets | keys): one
        # asynchronous host->device copy per stage(); the event guards reuse
        pin = (lambda t: t.pin_memory()) if torch.cuda.is_available() else (lambda t: t)
        self._pin_seeds = pin(torch.empty(nseed, dtype=torch.int32))
        self._pin_meta = pin(torch.empty(3 * self.max_nb + 1, dtype=torch.int64))
        self._pin_done = None
        self._fan = _lib.i32_array(self.fanouts.counts)
        ptr = lambda t: t.data_ptr() if t is not None else None
        self._out = _lib.FglSampleOut(
            ptr(self.tgt), ptr(self.src), ptr(self.wgt), e, ptr(self.tgt_row), ptr(self.src_row),
            ptr(self.tgt_front), ptr(self.src_front), ptr(self.unique), self.uniq_cap,
            ptr(self.frontier), self.fcap, ptr(self.seed_rows), ptr(self.seed_front),
            ptr(self.counts))

    def stage(self, seed_lists, seeds_for_rng):
        """Host->device copy of a window's seeds, offsets and Philox keys."""
        torch = self.torch
        nb = len(seed_lists)
        if nb < 1 or nb > self.max_nb:
            raise ValidationError(f"window of {nb} batches exceeds max_batches={self.max_nb}")
        sizes = [len(s) for s in seed_lists]
        if min(sizes) == 0:
            raise ValidationError("seeds must not be empty")
        if max(sizes) > self.max_bs:
            raise ValidationError("batch exceeds max_batch_size")
        off = np.zeros(nb + 1, dtype=np.int64)
        np.cumsum(sizes, out=off[1:])
        flat = np.concatenate([np.asarray(s) for s in seed_lists]).astype(np.int64)
        if flat.max() >= self.g.num_nodes or flat.min() < 0:
            raise ValidationError("seed id out of range")
        keys = np.array([philox_key(s) for s in seeds_for_rng], dtype=np.uint64).reshape(-1)
        n = int(off[-1])
        if self._pin_done is not None:
            from .trainer import _host_trace
            with _host_trace()("wait staging"):
                self._pin_done.synchronize()  # the previous window's copy has left the staging buffers
        self._pin_seeds.numpy()[:n] = flat
        meta = self._pin_meta.numpy()
        meta[: nb + 1] = off
        meta[nb + 1 : 3 * nb + 1] = keys.view(np.int64)
        self.seeds_dev[:n].copy_(self._pin_seeds[:n], non_blocking=True)
        self.seed_off[: nb + 1].copy_(self._pin_meta[: nb + 1], non_blocking=True)
        self.keys[: 2 * nb].copy_(self._pin_meta[nb + 1 : 3 * nb + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pin_done = ev
        return nb, off

    def run(self, nb: int, seed_off_host: np.ndarray, stream=None) -> DeviceWindow:
        """Launch the window sampler on staged inputs (asynchronous)."""
        st = stream if stream is not None else self.torch.cuda.current_stream()
        _lib.call("fgl_sample_window", self.g.struct, self.seeds_dev.data_ptr(),
                  self.seed_off.data_ptr(), int(seed_off_host[-1]), nb, self.keys.data_ptr(),
                  self._fan, self.H, self._out, self.ws.data_ptr(), self.ws_bytes, st.cuda_stream)
        if self.depth_layout:
            # rows of every batch in (depth, node id) order: each layer's rows become a prefix
            ws = self.ws.data_ptr()
            dc = self.counts.data_ptr() + 8 * counts_layout(self.H, nb)["len"]
            _lib.call("fgl_depth_relayout", self.counts.data_ptr(), self.H, nb, self.frontier.data_ptr(), self.fcap,
                      ws + self._bm_all_off, ws + self._prefix_off, self._words, self.unique.data_ptr(),
                      self.uniq_cap, self.tgt_row.data_ptr(), self.src_row.data_ptr(),
                      self.seed_rows.data_ptr(), int(seed_off_host[-1]), self.row_map.data_ptr(), dc,
                      self.relayout_ws.data_ptr(), self.relayout_ws.numel(), st.cuda_stream)
        return DeviceWindow(nb, self.H, self, seed_off_host)

    def sample(self, seed_lists, seeds_for_rng) -> DeviceWindow:
        nb, off = self.stage(seed_lists, seeds_for_rng)
        return self.run(nb, off)


_samplers: dict = {}


def _sampler_for(dg, fanouts, bs):
    key = (id(dg), tuple(fanouts))
    s = _samplers.get(key)
    if s is None or s.max_bs < bs or s.g is not dg:
        s = WindowSampler(dg, fanouts, max(bs, 1), 1)
        _samplers[key] = s
    return s


def sample_khop(g, seeds, fanouts, seed: int) -> SubgraphBatch:
    """K-hop uniform neighbor sampling; hop ``l`` uses ``fanouts.counts[l]``.

    Drop-in for sampler.py:120-139 (bit-exact, Philox(seed) stream)."""
    seeds = _validate_seeds(g.num_nodes, seeds)
    if not isinstance(fanouts, Fanouts):
        fanouts = Fanouts(fanouts)
    dg = device_graph(g)
    smp = _sampler_for(dg, fanouts.counts, len(seeds))
    win = smp.sample([seeds.astype(np.int64)], [seed])
    b = win.to_batch(0)
    b.seeds = seeds
    b.local_layers = []
    b.num_local = 0
    return b


class WalkSampler:
    """Device random-walk sampler (fgl_sample_walk) for batches of up to
    ``max_seeds`` seeds and walks of ``length`` steps; buffers are allocated
    once and results stay in HBM until the next call."""

    def __init__(self, dgraph, max_seeds: int, length: int, device="cuda"):
        import torch
        if length < 1:
            raise ValidationError("walk length must be >= 1")
        self.torch, self.g, self.length, self.max_seeds = torch, dgraph, int(length), int(max_seeds)
        e = self.max_seeds * self.length
        i32 = dict(dtype=torch.int32, device=device)
        self.tgt, self.src = torch.empty(e, **i32), torch.empty(e, **i32)
        self.wgt = torch.empty(e, dtype=torch.float32, device=device)
        self.step_off = torch.empty(self.length + 1, dtype=torch.int64, device=device)
        self.ucap = min(int(dgraph.num_nodes), self.max_seeds * (self.length + 1))
        self.unique = torch.empty(max(self.ucap, 1), **i32)
        self.counts = torch.zeros(2, dtype=torch.int64, device=device)
        self.seeds_dev = torch.empty(self.max_seeds, **i32)
        wsb = _lib.lib().fgl_walk_ws_bytes(dgraph.num_nodes, self.max_seeds)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=device)

    def run(self, seeds: np.ndarray, seed: int, stream=None):
        torch = self.torch
        n = len(seeds)
        if n > self.max_seeds:
            raise ValidationError("batch exceeds max_seeds")
        self.seeds_dev[:n].copy_(torch.from_numpy(np.asarray(seeds).astype(np.int32)))
        k0, k1 = philox_key(seed)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.call("fgl_sample_walk", self.g.struct, self.seeds_dev.data_ptr(), n, self.length, k0, k1,
                  self.tgt.data_ptr(), self.src.data_ptr(), self.wgt.data_ptr(), self.tgt.numel(),
                  self.step_off.data_ptr(), self.unique.data_ptr(), self.ucap, self.counts.data_ptr(),
                  self.ws.data_ptr(), self.ws.numel(), st)

    def to_batch(self, seeds: np.ndarray) -> SubgraphBatch:
        c = self.counts.cpu().numpy()
        _lib.status_error(int(c[1]), "fgl_sample_walk")
        ne = int(self.step_off[self.length].item())
        t = self.tgt[:ne].cpu().numpy().astype(np.uint64)
        s = self.src[:ne].cpu().numpy().astype(np.uint64)
        w = self.wgt[:ne].cpu().numpy()
        u = self.unique[: int(c[0])].cpu().numpy().astype(np.uint64)
        return SubgraphBatch(seeds=seeds, layers=[(t, s, w)], unique_nodes=u)


_WALKERS: dict = {}


def sample_random_walk(g, seeds, length: int, seed: int) -> SubgraphBatch:
    """One uniform random walk of ``length`` steps per seed; sinks stop early.

    Drop-in for sampler.py:142-186 (bit-exact, Philox(seed) stream): the walk
    runs as one GPU launch (fgl_sample_walk)."""
    seeds = _validate_seeds(g.num_nodes, seeds)
    if length < 1:
        raise ValidationError("walk length must be >= 1")
    dg = device_graph(g)
    key = (id(dg), int(length))
    ws = _WALKERS.get(key)
    if ws is None or ws.max_seeds < len(seeds):
        ws = WalkSampler(dg, max(len(seeds), 1024), length)
        _WALKERS[key] = ws
    ws.run(seeds, seed)
    return ws.to_batch(seeds)


def make_epoch_batches(g, train_ids, batch_size: int, shuffle_seed: int):
    """Seeded shuffle of the training IDs split into batches (sampler.py:189-198).
    Host-side (numpy Philox permutation); produces the seeds fed to the GPU."""
    if batch_size < 1:
        raise ValidationError("batch_size must be >= 1")
    train_ids = np.asarray(train_ids, dtype=np.uint64)
    if train_ids.size and train_ids.max() >= np.uint64(g.num_nodes):
        raise ValidationError("train id out of range")
    perm = np.random.Generator(np.random.Philox(shuffle_seed)).permutation(train_ids)
    return [perm[i : i + batch_size] for i in range(0, len(perm), batch_size)]
