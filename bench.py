#!/usr/bin/env python
"""Benchmark of the FastGL per-mini-batch hot path on B200 (BASELINE.json metric:
"epoch time & sampled edges/s (GCN, products-shape) at 1/2/4/8 B200").

A step is one Match-Reorder window of `window` mini-batches taken end to end:
Fused-Map sampling of the window, match-degree schedule, block-CSR prepare,
then per batch (in schedule order) Match delta feature load, forward, fp64
loss, backward, gradient all-reduce (N>1) and SGD.  `value` = sampled edges/s
of the whole job (all ranks), device-timed with CUDA events, max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config products]
    python bench.py --impl reference ...      # CPU oracle arm (rank 0 only)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "epoch time & sampled edges/s (GCN, products-shape) at 1/2/4/8 B200"
UNIT = "sampled edges/s"

CONFIGS = {
    # BASELINE.json configs[2] with the metric's model (GCN); the headline line
    "products": dict(
        desc="ogbn-products-shaped synthetic power-law graph (Chung-Lu, exponent 3, node IDs "
             "permuted), 2.45M nodes / 61.9M directed edges, 100-d f32 features resident in HBM, "
             "GCN (100,64,64,47), fanouts [15,10,5] (reference order: counts[0] expands the seeds), "
             "batch 1024, Match-Reorder window 8",
        nodes=2_450_000, edges=61_900_000, exponent=3.0, dims=(100, 64, 64, 47),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gcn", store="device"),
    "reddit": dict(
        desc="Reddit-shaped synthetic power-law graph (Chung-Lu), 233K nodes / 114.6M edges, "
             "602-d features in HBM, GCN (602,64,64,41), fanouts [15,10,5], batch 1024, window 8",
        nodes=233_000, edges=114_600_000, exponent=4.0, dims=(602, 64, 64, 41),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gcn", store="device"),
    "products_sage": dict(
        desc="products-shaped graph (BASELINE config 3 model), GraphSAGE-mean (1/indeg aggregation + root "
             "term, shared weight; SURVEY 8(c) extension) (100,64,64,47), fanouts [15,10,5], batch 1024, window 8",
        nodes=2_450_000, edges=61_900_000, exponent=3.0, dims=(100, 64, 64, 47),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="sage", store="device"),
    "gin": dict(
        desc="products-shaped graph, GIN 3-layer (100,64,64,47), fanouts [15,10,5], batch 1024, window 8",
        nodes=2_450_000, edges=61_900_000, exponent=3.0, dims=(100, 64, 64, 47),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gin", store="device"),
    "papers": dict(
        desc="ogbn-papers100M-shaped synthetic power-law graph (Chung-Lu, exponent 3), 111M nodes / "
             "1.6B directed edges, 128-d f32 features in PINNED HOST memory (Match-Reorder delta loads "
             "over the host link), GCN (128,64,64,172), fanouts [15,10,5], batch 1024, window 8",
        nodes=111_000_000, edges=1_600_000_000, exponent=3.0, dims=(128, 64, 64, 172),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gcn", store="host"),
    "products_host": dict(
        desc="products-shaped graph with the 100-d features in pinned host memory (Match delta "
             "loads over the host link), GCN (100,64,64,47), [15,10,5], batch 1024, window 8",
        nodes=2_450_000, edges=61_900_000, exponent=3.0, dims=(100, 64, 64, 47),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gcn", store="host"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML in a
    background thread every ~5 ms (the region is ~0.1 s), nvidia-smi -lms as
    the fallback."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.rows = []
        self.nvml = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self._stop = threading.Event()

            def run():
                while not self._stop.is_set():
                    try:
                        self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), int(get_reasons(h))))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.005)
            self._thr = threading.Thread(target=run, daemon=True)
            self._thr.start()
            return self
        except Exception:  # noqa: BLE001 - no NVML: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.nvml is not None:
            self._stop.set()
            self._thr.join(timeout=1)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if self.nvml is not None:
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": float(self.max_mhz), "reasons": ["unsampled"], "samples": 0}
            reasons = sorted({name for _, r in self.rows for bit, name in self.REASONS.items() if r & bit})
            return {"sm_mhz": statistics.median(float(c) for c, _ in self.rows), "sm_max_mhz": float(self.max_mhz),
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml"}
        rows = []
        for line in (getattr(self, "out", "") or "").splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


# ---------------------------------------------------------------- workload --
def build_workload(cfg, device):
    import torch
    from paper_2409_14939_b200.graph import chung_lu_graph
    t0 = time.time()
    dg = chung_lu_graph(cfg["nodes"], cfg["edges"], exponent=cfg["exponent"], seed=0, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(1)
    feats = torch.randn((dg.num_nodes, cfg["dims"][0]), generator=gen, device=device, dtype=torch.float32)
    labels = torch.randint(0, cfg["dims"][-1], (dg.num_nodes,), generator=gen, device=device)
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    log(f"graph: {dg.num_nodes} nodes, {dg.num_edges} edges, max degree "
        f"{int((dg.row_offsets[1:] - dg.row_offsets[:-1]).max())}; built in {time.time() - t0:.1f}s")
    return dg, feats, labels


def epoch_windows(num_nodes, cfg, seed=0):
    from paper_2409_14939_b200.sampler import derive_seed
    rng = np.random.Generator(np.random.Philox(derive_seed(seed, 7)))
    perm = rng.permutation(num_nodes)
    train_ids = perm[: max(1, int(0.8 * num_nodes))]
    shuf = np.random.Generator(np.random.Philox(derive_seed(seed, 11))).permutation(train_ids)
    bs = cfg["bs"]
    batches = [shuf[i : i + bs] for i in range(0, len(shuf), bs)]
    nwin = cfg["window"]
    wins = []
    for w0 in range(0, len(batches), nwin):
        wb = batches[w0 : w0 + nwin]
        if len(wb) == nwin and all(len(b) == bs for b in wb):  # full windows only (equal steps per rank)
            wins.append(([b.astype(np.int64) for b in wb], [derive_seed(seed, 13, w0 + j) for j in range(nwin)]))
    return wins, len(batches)


# ------------------------------------------------------------- cpu oracle --
_CPU = {}


def _cpu_batch(args):
    import oracle
    seeds, rs = args
    g, feats, labels, dims, fanouts, arch, params = (_CPU[k] for k in
                                                     ("g", "feats", "labels", "dims", "fanouts", "arch", "params"))
    t0 = time.perf_counter()
    b = oracle.sample_khop(g, seeds, fanouts, rs)
    p = [[w.copy(), bb.copy()] for w, bb in params]
    oracle.train_step(b, feats, labels, p, 0.1, arch)
    return b.num_sampled_edges(), time.perf_counter() - t0


def cpu_oracle_throughput(dg, feats, labels, cfg, windows, budget_s=25.0, workers=None):
    """Reference algorithm (oracle port of sample_khop + _prepare_batch + forward/
    backward/SGD, trainer.py:301-323) on the host cores, one mini-batch per
    worker process; returns (edges/s, cores, sample description)."""
    import multiprocessing as mp

    import oracle
    from paper_2409_14939_b200.graph import to_host
    hg = to_host(dg)
    g = oracle.CSRGraph(hg.num_nodes, hg.row_offsets, hg.col_indices, None, None, None)
    _CPU.update(g=g, feats=feats.cpu().numpy(), labels=labels.cpu().numpy(), dims=cfg["dims"],
                fanouts=cfg["fanouts"], arch=cfg["arch"], params=oracle.init_params(cfg["dims"], 0))
    workers = workers or max(1, min(os.cpu_count() or 1, 16))
    # one probe batch sizes the sample to the time budget
    seeds, rs = windows[0][0][0], windows[0][1][0]
    e0, t_one = _cpu_batch((seeds, rs))
    # batches run ~2-3x slower when all workers share the host; keep the
    # sample near the budget
    per_worker = max(1, int(budget_s // max(3.0 * t_one, 1e-3)))
    per_worker = min(per_worker, 4)
    jobs = []
    for w_seeds, w_rs in windows:
        for s, r in zip(w_seeds, w_rs):
            jobs.append((s, r))
            if len(jobs) >= workers * per_worker:
                break
        if len(jobs) >= workers * per_worker:
            break
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_cpu_batch, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    edges = sum(r[0] for r in res)
    sample = (f"{len(jobs)} mini-batches of the same workload (oracle port of the reference per-batch "
              f"pipeline: sample_khop, _prepare_batch, x0 gather, forward, fp64 loss, backward, SGD), "
              f"{workers} worker processes, {wall:.1f}s wall; single batch {t_one:.1f}s")
    return edges / wall, workers, sample, wall


# ------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="products", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--profile", action="store_true", help="stop after warm-up + 2 steps (for ncu)")
    ap.add_argument("--cache-ratio", type=float, default=0.0,
                    help="static-degree HBM feature cache in front of a host-resident store (configs *_host, papers)")
    args = ap.parse_args()

    import torch
    from paper_2409_14939_b200 import dist as fdist
    cfg = CONFIGS[args.config]
    rank, world = fdist.init("nccl") if int(os.environ.get("WORLD_SIZE", "1")) > 1 else (0, 1)
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world, local)
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    from paper_2409_14939_b200 import _lib, trainer

    dg, feats, labels = build_workload(cfg, device)
    windows, nbatches = epoch_windows(dg.num_nodes, cfg)
    mine = fdist.shard(windows, rank, world)
    mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch=cfg["arch"],
                               batch_size=cfg["bs"], window_n=cfg["window"], lr=0.1, seed=0)
    pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device=device,
                            feature_store=cfg["store"], dist=fdist.GradAllReduce(world),
                            direct_x0=cfg.get("direct_x0", True),
                            cache_ratio=args.cache_ratio if cfg["store"] == "host" else 0.0)
    lib = _lib.lib()
    W, K = max(args.warmup, 0), max(args.steps, 1)
    if args.profile:
        W, K = max(W, 1), 2
    it = 0

    def take(n):
        nonlocal it
        out = [mine[(it + k) % len(mine)] for k in range(n)]
        it += n
        return out

    # sampling of window w+1 overlaps the compute of window w (Pipeline.run_windows)
    for _ in pipe.run_windows(take(W)):
        pass
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # ---------------- timed region (device time, CUDA events on the stream) --
    edges = 0
    draws = 0
    l0 = lib.fgl_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if args.profile:  # ncu --profile-from-start off: capture only the timed steps
            torch.cuda.profiler.start()
        ev0.record()
        for _ in pipe.run_windows(take(K)):
            win = pipe.last_window
            edges += win.total_edges()
            draws += sum(win.draws(b) for b in range(win.num_batches))
        ev1.record()
        torch.cuda.synchronize()
        if args.profile:
            torch.cuda.profiler.stop()
    launches = lib.fgl_launch_count() - l0
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = fdist.max_over_ranks(ms, world, device)
    edges_all = fdist.sum_over_ranks(float(edges), world, device)
    value = edges_all / (ms_max / 1e3)
    ms_per_step = ms_max / K
    batches_per_step = cfg["window"] * world
    epoch_s = nbatches / batches_per_step * ms_per_step / 1e3

    if args.profile:  # launch-list / ncu runs: the timed steps are all that is needed
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step}), flush=True)
        return
    # ---------------- stage breakdown + roofline (instrumented extra steps) --
    stages = stage_profile(pipe, mine, it, cfg, torch)
    it += 2
    # ---------------- end to end through the public API with host buffers ----
    e2e = e2e_measure(pipe, mine, it, K, torch, world, device)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 loss; int32/int64 sampling)",
        "data": "synthetic (seeded Chung-Lu power-law graph, random f32 features, random labels)",
        "config": {"workload": cfg["desc"] + (f", static-degree HBM cache ratio {args.cache_ratio}"
                                              if args.cache_ratio and cfg["store"] == "host" else ""),
                   "global_batch": cfg["bs"] * world,
                   "windows_per_step_per_rank": 1, "mini_batches_per_step": batches_per_step,
                   "parallelism": f"dp{world}", "l2": "inputs (CSR 0.27 GB + features) larger than the 126 MB L2",
                   "epoch_batches": nbatches},
        "epoch_time_s": epoch_s,
        "sampled_edges_per_step": edges_all / K,
        "philox_draws_per_step": fdist.sum_over_ranks(float(draws), world, device) / K,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "stages_ms_per_step": stages["ms"],
        "roofline": stages["roofline"],
        "e2e": e2e,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        v, cores, sample, wall = cpu_oracle_throughput(dg, feats, labels, cfg, mine, args.cpu_budget)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def _measured_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture
    of `kernel` (same workload, committed under profiles/), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel, {}).get("traffic_bytes")
    except Exception:
        return None


def stage_profile(pipe, mine, it, cfg, torch):
    """Per-stage device time of 2 windows (events between the stages; not part
    of the headline timing) and the roofline of the dominant stage."""
    import json as _json
    peaks = _json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    acc = {"sample": 0.0, "schedule": 0.0, "prepare": 0.0, "compute": 0.0}
    draws = 0
    samp_bytes = 0.0
    from paper_2409_14939_b200 import _lib as _l
    sel = {"s": 0.0, "bytes": 0.0, "draws": 0.0}
    pipe.loaded.zero_()
    pipe.cache_hits.zero_()
    for k in range(2):
        seeds, rs = mine[(it + k) % len(mine)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        _l.call("fgl_profile_select", 1)
        ev[0].record()
        win = pipe.sampler.sample(seeds, rs)
        ev[1].record()
        _l.call("fgl_profile_select", 0)
        pms = np.zeros(16, dtype=np.float64)
        nl = np.zeros(1, dtype=np.int64)
        _l.call("fgl_profile_select_read", pms.ctypes.data, 16, nl.ctypes.data)
        win.host_counts()
        order = pipe.schedule(win, len(seeds))
        ev[2].record()
        layers = pipe.prepare(win)
        ev[3].record()
        for j, b in enumerate(order):
            pipe.batch_step(win, b, order[j - 1] if j else None, j, layers, j % 2)
        ev[4].record()
        torch.cuda.synchronize()
        for i, name in enumerate(acc):
            acc[name] += ev[i].elapsed_time(ev[i + 1]) / 2
        nb = win.num_batches
        draws += sum(win.draws(b) for b in range(nb)) / 2
        # algorithmic sampler bytes: offsets of each frontier node,
        # chosen col (+weight) reads, (t, s, w) writes
        for h in range(win.num_hops):
            F = win.front_total(h)
            e0, e1 = win.hop_edges(h)
            S = e1 - e0
            samp_bytes += (2 * 8 * F + S * 4 + S * (2 * 4 + 4)) / 2
        # dominant launch: the last hop's select kernel (largest frontier).
        # Algorithmic bytes: per frontier node its id, batch, two CSR offsets,
        # the two scans (4+4+16+16); per sampled edge the chosen col entry and
        # the (tgt, src, wgt, tgt_front) record (4 + 16); draws: one per candidate
        hl = win.num_hops - 1
        F = win.front_total(hl)
        e0_, e1_ = win.hop_edges(hl)
        S = e1_ - e0_
        sel["s"] += float(pms[hl]) / 1e3 / 2
        sel["bytes"] += (40.0 * F + 20.0 * S) / 2
        sel["draws"] += win.hop_draws(hl) / 2
    t_s = acc["sample"] / 1e3
    # Philox ALU probe: draws/s of the bare Philox4x64-10 kernel on this GPU
    from paper_2409_14939_b200 import _lib
    buf = torch.empty(148 * 8 * 256, dtype=torch.int64, device=pipe.device)
    nblk = 1 << 27
    _lib.call("fgl_philox_bench", 1, 2, nblk, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("fgl_philox_bench", 3, 4, nblk, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    peak_draws = 4 * nblk / (e0.elapsed_time(e1) / 1e3)
    roof = {
        "kernel": "select_bal_kernel + select_hub_kernel (hop-2 selection of fgl_sample_window, the largest select launch)",
        "bound": "hbm", "achieved": sel["bytes"] / sel["s"] / 1e9, "peak": hbm_peak, "unit": "GB/s",
        "frac": sel["bytes"] / sel["s"] / 1e9 / hbm_peak, "traffic": _measured_traffic("select_bal_kernel"),
        "peak_source": peak_src, "launch_ms": sel["s"] * 1e3, "bytes_per_launch": sel["bytes"],
        "alu": {"bound": "philox4x64-10 draws (bit-exact sampling needs one per candidate edge)",
                "achieved_draws_per_s": sel["draws"] / sel["s"], "peak_draws_per_s": peak_draws,
                "frac": sel["draws"] / sel["s"] / peak_draws,
                "draws_per_launch": sel["draws"]},
        "sampler_stage": {"ms_per_window": acc["sample"], "draws_per_s": draws / t_s,
                          "alu_frac": draws / t_s / peak_draws},
    }
    if pipe.feature_store == "host":
        # IO stage: feature rows that cross the host link per
        # window vs the measured pinned host->device copy peak of this box
        loaded = int(pipe.loaded.item()) / 2
        hits = int(pipe.cache_hits.item()) / 2
        link_bytes = loaded * 4 * pipe.d0
        hb = torch.empty(1 << 28, dtype=torch.float32).pin_memory()
        db = torch.empty(1 << 28, dtype=torch.float32, device=pipe.device)
        db.copy_(hb, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        db.copy_(hb, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        link_peak = hb.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
        del hb, db
        achieved = link_bytes / (acc["compute"] / 1e3) / 1e9
        roof["io"] = {"bound": "host link (pinned zero-copy row gathers)", "rows_per_window": loaded,
                      "cache_rows_per_window": hits, "bytes_per_window": link_bytes,
                      "achieved": achieved, "peak": link_peak, "unit": "GB/s", "frac": achieved / link_peak,
                      "peak_source": "measured: pinned host->device cudaMemcpy of 1 GiB on this box",
                      "note": "achieved = host-link bytes / whole compute stage time (lower bound for the gather)"}
    return {"ms": acc, "roofline": roof}


def e2e_measure(pipe, mine, it, K, torch, world, device):
    """Same metric through the public API with host buffers: each step stages
    the window's seeds from pinned host memory (H2D inside the timed region)
    and copies its per-batch losses back to pinned host memory (D2H inside the
    timed region, asynchronous); wall clock (synchronised), max over ranks."""
    from paper_2409_14939_b200 import dist as fdist
    edges = 0
    h2d = d2h = 0
    staged = []
    for k in range(K):  # the caller's inputs live in pinned host memory before the clock starts
        seeds, rs = mine[(it + k) % len(mine)]
        pinned = [torch.from_numpy(s.astype(np.int64)).pin_memory() for s in seeds]
        staged.append(([p.numpy() for p in pinned], rs))
        h2d += sum(len(s) for s in seeds) * 4 + (len(seeds) + 1) * 8 + 16 * len(seeds)
    host_losses = [torch.empty(len(staged[k][0]), dtype=torch.float64).pin_memory() for k in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, (order, losses) in enumerate(pipe.run_windows(staged)):
        # per-batch losses of every step copied back to pinned host memory
        # (asynchronous D2H on the compute stream; no per-step host stall)
        host_losses[k].copy_(losses, non_blocking=True)
        edges += pipe.last_window.total_edges()
        d2h += host_losses[k].numel() * 8
    torch.cuda.synchronize()
    _ = [float(h.sum()) for h in host_losses]  # the host consumes every step's losses
    wall = time.perf_counter() - t0
    wall = fdist.max_over_ranks(wall, world, device)
    edges_all = fdist.sum_over_ranks(float(edges), world, device)
    return {"value": edges_all / wall, "unit": UNIT, "h2d_bytes_per_step": h2d // K,
            "d2h_bytes_per_step": d2h // K}


def cpu_reference_steps(dg, feats, labels, cfg, windows, steps, warmup, budget_s):
    """Reference arm in steps: one step = one mini-batch per host worker
    process, all workers in parallel (oracle port of the reference per-batch
    pipeline).  `warmup` untimed rounds, then up to `steps` timed rounds --
    fewer if they would exceed `budget_s` (CPU batches take seconds each)."""
    import multiprocessing as mp

    import oracle
    from paper_2409_14939_b200.graph import to_host
    hg = to_host(dg)
    g = oracle.CSRGraph(hg.num_nodes, hg.row_offsets, hg.col_indices, None, None, None)
    _CPU.update(g=g, feats=feats.cpu().numpy(), labels=labels.cpu().numpy(), dims=cfg["dims"],
                fanouts=cfg["fanouts"], arch=cfg["arch"], params=oracle.init_params(cfg["dims"], 0))
    workers = max(1, min(os.cpu_count() or 1, 16))
    jobs = [(s, r) for w_seeds, w_rs in windows for s, r in zip(w_seeds, w_rs)]
    k = 0

    def take():
        nonlocal k
        out = [jobs[(k + i) % len(jobs)] for i in range(workers)]
        k += workers
        return out

    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        t_round = None
        for _ in range(max(1, min(warmup, 2))):  # the first round also forks / warms the workers
            t0 = time.perf_counter()
            pool.map(_cpu_batch, take(), chunksize=1)
            t_round = time.perf_counter() - t0
        rounds = max(1, min(steps, int(budget_s // max(t_round, 1e-3))))
        edges, t0 = 0, time.perf_counter()
        for _ in range(rounds):
            edges += sum(r[0] for r in pool.map(_cpu_batch, take(), chunksize=1))
        wall = time.perf_counter() - t0
    sample = (f"{rounds} timed rounds x {workers} mini-batches (one per worker process, in parallel) of the "
              f"same workload, oracle port of the reference per-batch pipeline (sample_khop, _prepare_batch, "
              f"x0 gather, forward, fp64 loss, backward, SGD); {wall:.1f}s wall")
    return edges / wall, workers, sample, wall, rounds


def run_reference(args, cfg, rank, world, local):
    """CPU reference arm: the oracle port of the reference's per-batch pipeline on
    the host cores (rank 0 only); same workload, metric and unit."""
    if rank != 0:
        return
    import torch
    has_gpu = torch.cuda.is_available()
    device = f"cuda:{local}" if has_gpu else "cpu"
    dg, feats, labels = build_workload(cfg, device)
    windows, nbatches = epoch_windows(dg.num_nodes, cfg)
    v, cores, sample, wall, rounds = cpu_reference_steps(dg, feats, labels, cfg, windows, max(args.steps, 1),
                                                         max(args.warmup, 0), args.cpu_budget)
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": rounds,
        "steps_requested": args.steps, "warmup": max(1, min(args.warmup, 2)),
        "ms_per_step": wall / rounds * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "impl": "reference", "dtype": "f32 (fp64 loss)", "data": "synthetic",
        "config": {"workload": cfg["desc"], "global_batch": cfg["bs"], "parallelism": f"{cores} cpu processes"},
        "epoch_time_s": None,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
