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
import gc
import json
import os

# every kernel module loaded at context creation, not at its first launch
# inside a timed region (lazy loading from a cold page cache on a fresh box)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
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
    "papers_hbm": dict(
        desc="ogbn-papers100M-shaped synthetic power-law graph (Chung-Lu, exponent 3), 111M nodes / "
             "1.6B directed edges, 128-d f32 features RESIDENT IN HBM (56.8 GB of the B200's 180 GB: the "
             "B200-native placement of config 4; layer 0 reads the table directly), GCN (128,64,64,172), "
             "fanouts [15,10,5], batch 1024, window 8",
        nodes=111_000_000, edges=1_600_000_000, exponent=3.0, dims=(128, 64, 64, 172),
        fanouts=[15, 10, 5], bs=1024, window=8, arch="gcn", store="device"),
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


def _host_features(feats, cfg):
    """[N, d] host array of the workload's features (a view for a pinned store)."""
    table = getattr(feats, "table", None)
    if table is not None:
        return table[:, : cfg["dims"][0]].numpy()
    return feats.cpu().numpy()


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
    _CPU.update(g=g, feats=_host_features(feats, cfg), labels=labels.cpu().numpy(), dims=cfg["dims"],
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
def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: launch the N ranks (one
    process per GPU, NCCL over NVLink) through torch.distributed.run on
    127.0.0.1 and return its exit code; rank 0 prints the JSON line."""
    import torch
    if args.impl == "ours" and args.dist_backend == "nccl" and torch.cuda.device_count() < args.gpus:
        log(f"bench: --gpus {args.gpus} needs {args.gpus} visible GPUs for NCCL (found {torch.cuda.device_count()}); "
            f"--dist-backend gloo runs the ranks on fewer GPUs (functional check, not a measurement)")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ)
    if args.impl == "ours" and args.dist_backend == "nccl":
        # the communicator's INIT lines (rings / NVLS / channels) on stderr
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    log("bench: spawning", " ".join(cmd))
    return subprocess.call(cmd, env=env)


def make_feature_store(cfg, dg, rank, world, device):
    """BASELINE config 4: the feature table in pinned HOST memory, ONE copy
    for all ranks of the node (HostFeatureStore.shared: rank 0 fills a
    shared-memory table that every rank maps and page-locks).  Rank 0
    generates the rows on its GPU chunk by chunk (seeded)."""
    import torch
    from paper_2409_14939_b200.store import HostFeatureStore
    n, d = dg.num_nodes, cfg["dims"][0]

    def fill(table):
        gen = torch.Generator(device=device)
        gen.manual_seed(1)
        chunk = 1 << 22
        for i in range(0, n, chunk):
            m = min(chunk, n - i)
            table[i : i + m, :d].copy_(torch.randn((m, d), generator=gen, device=device, dtype=torch.float32).cpu())
    t0 = time.time()
    st = HostFeatureStore.shared(n, d, fill, rank=rank, world=world)
    log(f"rank {rank}: shared pinned feature store {n} x {st.ld} f32 ({n * st.ld * 4 / 2**30:.1f} GiB, "
        f"one copy for {world} rank(s)) ready in {time.time() - t0:.1f}s")
    return st


def config_dict(cfg, args, world, nbatches):
    """The `config` object of both arms (same keys, same workload string)."""
    return {"workload": cfg["desc"] + (f", static-degree HBM cache ratio {args.cache_ratio}"
                                       if args.cache_ratio and cfg["store"] == "host" else ""),
            "batch_size": cfg["bs"], "global_batch": cfg["bs"] * world,
            "windows_per_step_per_rank": 1, "mini_batches_per_step": cfg["window"] * world,
            "parallelism": f"dp{world}" + ("" if world == 1 else f" ({args.dist_backend})"),
            "l2": "inputs (CSR 0.27 GB + features) larger than the 126 MB L2",
            "epoch_batches": nbatches}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="products", choices=sorted(CONFIGS))
    ap.add_argument("--bs", type=int, default=0, help="batch size override (config 5 sweep: 512..8192)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share a GPU (functional check of the N-rank path, not a measurement)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--profile", action="store_true", help="stop after warm-up + 2 steps (for ncu)")
    ap.add_argument("--cache-ratio", type=float, default=0.0,
                    help="static-degree HBM feature cache in front of a host-resident store (configs *_host, papers)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    import torch
    from paper_2409_14939_b200 import dist as fdist
    cfg = dict(CONFIGS[args.config])
    if args.bs:
        cfg["bs"] = int(args.bs)
        cfg["desc"] = cfg["desc"].replace("batch 1024", f"batch {args.bs}")
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":  # CPU arm: rank 0 alone, no process group
        return run_reference(args, cfg, int(os.environ.get("RANK", 0)), world_env, local)
    rank, world = fdist.init(args.dist_backend) if world_env > 1 else (0, 1)
    torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
    device = f"cuda:{torch.cuda.current_device()}"
    from paper_2409_14939_b200 import _lib, trainer

    if cfg["store"] == "host":
        from paper_2409_14939_b200.graph import chung_lu_graph
        dg = chung_lu_graph(cfg["nodes"], cfg["edges"], exponent=cfg["exponent"], seed=0, device=device)
        feats = make_feature_store(cfg, dg, rank, world, device)
        gen = torch.Generator(device=device)
        gen.manual_seed(2)
        labels = torch.randint(0, cfg["dims"][-1], (dg.num_nodes,), generator=gen, device=device)
    else:
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
    fb0 = lib.fgl_dense_fallback_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the host feeds the pipeline: a garbage-collector pause inside a timed
    # region stalls the device too (one GIN run read 0.74G e2e vs 1.63G), so
    # collect up front and keep the collector off while timing
    gc.collect()
    gc.disable()
    with ClockSampler(torch.cuda.current_device()) as clk:
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
    fallbacks = lib.fgl_dense_fallback_count() - fb0
    if fallbacks:
        raise RuntimeError(f"{fallbacks} dense layers ran on the SIMT fallback inside the timed region")
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
        gc.enable()
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step}), flush=True)
        return
    # ---------------- per-stage rooflines (live, instrumented extra steps) ----
    stages = stage_profile(pipe, take(4), cfg, torch)
    # ---------------- end to end through the public API with host buffers ----
    e2e_measure(pipe, take(min(K, 3)), torch, world, device)  # untimed: first use of the host-buffer path
    gc.collect()
    e2e = e2e_measure(pipe, take(K), torch, world, device)
    gc.enable()

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 loss; int32/int64 sampling)",
        "data": "synthetic (seeded Chung-Lu power-law graph, random f32 features, random labels)",
        "config": config_dict(cfg, args, world, nbatches),
        "epoch_time_s": epoch_s,
        "sampled_edges_per_step": edges_all / K,
        "philox_draws_per_step": fdist.sum_over_ranks(float(draws), world, device) / K,
        "gpu_launches": int(launches),
        "dense_fallbacks": int(fallbacks),
        "clocks": clk.summary(),
        "stages_ms_per_step": stages["ms"],
        "roofline": stages["roofline"],
        "stage_rooflines": stages["stages"],
        "e2e": e2e,
    }
    if world > 1:
        out["allreduce"] = allreduce_probe(pipe, torch, world, device)
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


_TRAFFIC_KEYS = {"select": "select_bal2_kernel", "aggregate_l0": "spmm_lean_kernel_l0",
                 "dense_fwd": "tc_dense4_kernel_l0", "wgrad": "tc_wgrad3_kernel_l0", "gather": "gather_rows_kernel_host"}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(p.read_text()) if p.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6540.8))
    bf16 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1328.6)))
    src = "MEASURED_PEAKS.json (driver-measured copy bandwidth / cuBLAS bf16, sustained)" if peaks else \
        "fallback figures of B200_PROFILING.md"
    return hbm, bf16, src


def philox_peak(torch, device):
    """Measured Philox4x64-10 throughput of this GPU (draws/s): the bare
    counter-based generator with nothing else (fgl_philox_bench: full
    occupancy, per-lane keys as in the select kernels)."""
    from paper_2409_14939_b200 import _lib
    buf = torch.empty(148 * 8 * 256, dtype=torch.int64, device=device)
    nblk = 1 << 27
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("fgl_philox_bench", 1, 2, nblk, buf.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("fgl_philox_bench", 3, 4, nblk, buf.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    threads = 148 * 8 * 256
    return 4 * (nblk // threads) * threads / (e0.elapsed_time(e1) / 1e3)


def host_link_peak(torch, device):
    hb = torch.empty(1 << 28, dtype=torch.float32).pin_memory()
    db = torch.empty(1 << 28, dtype=torch.float32, device=device)
    db.copy_(hb, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.copy_(hb, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return hb.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9


def _roof(bound, achieved, peak, unit, traffic_key=None, **extra):
    out = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak if peak else None,
           "traffic": _measured_traffic(_TRAFFIC_KEYS.get(traffic_key, traffic_key)) if traffic_key else None}
    out.update(extra)
    return out


def stage_profile(pipe, wins, cfg, torch):
    """Per-stage rooflines from LIVE kernel times: the timed pipeline itself
    (run_windows: CUDA graphs; sampling, prepare / layer-0 aggregation and
    the model chain on their concurrent streams) runs extra windows with
    fgl_profile on, so the library brackets its dominant launches with CUDA
    events on their own streams (event-record nodes inside the graphs, timed
    on every replay).  Each stage's achieved
    rate = its ALGORITHMIC bytes or draws over those launches
    / their summed device time; `bound` is the roof with the larger fraction.
    The headline `roofline` is the stage whose kernels take the most device
    time."""
    import ctypes

    from paper_2409_14939_b200 import _lib
    lib = _lib.lib()
    hbm_peak, bf16_peak, peak_src = _peaks()
    tf32_peak = bf16_peak / 2  # dense tf32 rate of the tensor cores = half of bf16 (3xTF32 issues 3 MMAs)
    device = pipe.device
    d0 = cfg["dims"][0]
    H = len(cfg["fanouts"])
    weighted = pipe.dg.edge_weights is not None
    pipe.loaded.zero_()
    pipe.cache_hits.zero_()
    hop = {h: {"F": 0, "S": 0} for h in range(H)}
    l0 = {"n": 0, "E": 0, "launches": 0}
    torch.cuda.synchronize()
    lib.fgl_profile(1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    draws_total = 0
    try:
        for _ in pipe.run_windows(wins):
            win = pipe.last_window
            for h in range(H):  # host counts only: no device sync inside the loop
                e0, e1 = win.hop_edges(h)
                hop[h]["F"] += win.front_total(h)
                hop[h]["S"] += e1 - e0
            draws_total += sum(win.draws(b) for b in range(win.num_batches))
            e0, e1 = win.hop_edges(H - 1)
            l0["E"] += e1 - e0
            l0["launches"] += win.num_batches
        ev1.record()
        torch.cuda.synchronize()
    finally:
        lib.fgl_profile(0)
    loaded = int(pipe.loaded.sum().item())
    cap = 1 << 16
    ids = np.zeros(cap, np.int32)
    args3 = np.zeros(3 * cap, np.int64)
    ms = np.zeros(cap, np.float64)
    cnt = ctypes.c_int64()
    _lib.call("fgl_profile_read", cap, ids.ctypes.data, args3.ctypes.data, ms.ctypes.data, ctypes.byref(cnt))
    k = min(int(cnt.value), cap)
    ids, args3, ms = ids[:k], args3[: 3 * k].reshape(k, 3), ms[:k]
    nwin = len(wins)
    window_ms = ev0.elapsed_time(ev1) / nwin

    def tot(mask):
        return float(ms[mask].sum()) / 1e3, int(mask.sum())

    stages = {}
    # --- sample: select_bal + select_hub per hop; INT-ALU (Philox) and HBM roofs
    t, n = tot(ids == 1)
    if n:
        draws = draws_total
        bytes_ = sum(2 * 8 * v["F"] + v["S"] * (4 + 4 * weighted) + v["S"] * (2 * 4 + 4) for v in hop.values())
        peak_draws = philox_peak(torch, device)
        alu = draws / t / peak_draws
        hbmf = bytes_ / t / 1e9 / hbm_peak
        stages["sample"] = _roof("alu" if alu >= hbmf else "hbm", draws / t, peak_draws, "draws/s", "select",
                                 kernel="select_bal_kernel + select_hub_kernel (every hop)", launches=n,
                                 ms_per_window=t * 1e3 / nwin, draws_per_launch=draws / n,
                                 hbm={"achieved": bytes_ / t / 1e9, "peak": hbm_peak, "unit": "GB/s", "frac": hbmf,
                                      "bytes_per_launch": bytes_ / n,
                                      "model": "SURVEY 8(d): 16 B offsets per frontier node, chosen col (+w) read, "
                                               "(t, s, w) written per sampled edge"},
                                 peak_source="measured: fgl_philox_bench, bare Philox4x64-10 on this GPU")
    # --- layer-0 aggregation (the largest SpMM): HBM, reference byte model
    agg_id = 2 if (ids == 2).any() else 3
    mask = (ids == agg_id) & (args3[:, 1] == d0)
    t, n = tot(mask)
    if n:
        rows = int(args3[mask, 0].sum())
        E = l0["E"] if agg_id == 2 or n == l0["launches"] else None
        if E is not None:
            bytes_ = 8 * (rows + n) + E * (4 + 4) + 4 * E * d0 + 4 * rows * d0
            stages["aggregate_l0"] = _roof(
                "hbm", bytes_ / t / 1e9, hbm_peak, "GB/s", "aggregate_l0",
                kernel="spmm_lean_kernel (fgl_spmm_gather)" if agg_id == 2 else "fgl_spmm (layer-0 rows)",
                launches=n, ms_per_window=t * 1e3 / nwin, bytes_per_launch=bytes_ / n,
                model="memsim.py:96 / Eq. 3: 8(n+1) + E(4+4) + 4 E d + 4 n d", peak_source=peak_src,
                flops_per_launch=2 * E * d0 / n)
    # --- dense forward / dgrad / weight gradient: HBM (intensity below the ridge); tensor pipe reported
    for name, pid, byte_fn, flop_fn, kname in [
            ("dense_fwd", 4, lambda M, N, K: 4 * (M * K + K * N + 2 * M * N), lambda M, N, K: 2 * M * N * K,
             "tc_dense4_kernel<0> (all layers; tc_gemm3 for K slices)"),
            ("dgrad", 5, lambda M, N, K: 4 * (2 * M * K + K * N + M * N), lambda M, N, K: 2 * M * N * K,
             "tc_dense4_kernel<1> (all layers; tc_gemm3 for K slices)"),
            ("wgrad", 6, lambda M, K, N: 4 * (M * K + 2 * M * N), lambda M, K, N: 2 * M * K * N,
             "tc_wgrad3_kernel + reduce_partials (all layers)")]:
        mask = ids == pid
        t, n = tot(mask)
        if not n:
            continue
        a = args3[mask]
        bytes_ = float(sum(byte_fn(*map(int, r)) for r in a))
        flops = float(sum(flop_fn(*map(int, r)) for r in a))
        stages[name] = _roof("hbm", bytes_ / t / 1e9, hbm_peak, "GB/s", name if name != "dgrad" else None,
                             kernel=kname, launches=n, ms_per_window=t * 1e3 / nwin, bytes_per_launch=bytes_ / n,
                             tensor={"achieved_tflops": flops / t / 1e12, "peak_tflops": tf32_peak,
                                     "frac": flops / t / 1e12 / tf32_peak,
                                     "note": "fp32-accurate 3xTF32: 3 tf32 MMAs per product; peak = dense tf32 "
                                             "(half of the measured bf16)"},
                             peak_source=peak_src)
    # --- IO: x0 rows over the host link (host-resident feature store)
    mask = ids == 7
    t, n = tot(mask)
    if n and pipe.feature_store == "host":
        link = host_link_peak(torch, device)
        link_bytes = loaded * 4 * d0
        stages["io"] = _roof("host_link", link_bytes / t / 1e9, link, "GB/s", "gather",
                             kernel="gather_rows_kernel (Match delta + cache + zero-copy host rows)", launches=n,
                             ms_per_window=t * 1e3 / nwin, rows_per_window=loaded / nwin,
                             bytes_per_launch=link_bytes / n,
                             peak_source="measured: pinned host->device cudaMemcpy of 1 GiB on this box")
    per_stage_ms = {k: v["ms_per_window"] for k, v in stages.items()}
    per_stage_ms["window"] = window_ms
    names = {1: "select", 2: "aggregate_l0 (fgl_spmm_gather)", 3: "fgl_spmm (other aggregations incl. transposed)",
             4: "dense_fwd", 5: "dgrad", 6: "wgrad", 7: "x0 gather", 8: "top layer", 9: "sgd"}
    per_stage_ms["kernels"] = {names.get(int(i), str(int(i))): {"ms_per_window": float(ms[ids == i].sum()) / nwin,
                                                                "launches_per_window": int((ids == i).sum()) / nwin}
                               for i in np.unique(ids)}
    dom = max(stages, key=lambda k: stages[k]["ms_per_window"]) if stages else None
    head = dict(stages[dom]) if dom else {}
    if head:
        head["stage"] = dom
        head["why_dominant"] = (f"largest summed device time of the profiled launches per window "
                                f"({head['ms_per_window']:.3f} ms); live times (graph replays, concurrent streams)")
    return {"ms": per_stage_ms, "roofline": head, "stages": stages}


def e2e_measure(pipe, wins, torch, world, device):
    """Same metric through the public API with host buffers: each step stages
    the window's seeds from pinned host memory (H2D inside the timed region)
    and copies its per-batch losses back to pinned host memory (D2H inside the
    timed region, asynchronous); wall clock (synchronised), max over ranks."""
    from paper_2409_14939_b200 import dist as fdist
    edges = 0
    h2d = d2h = 0
    staged = []
    K = len(wins)
    for seeds, rs in wins:  # the caller's inputs live in pinned host memory before the clock starts
        pinned = [torch.from_numpy(s.astype(np.int64)).pin_memory() for s in seeds]
        staged.append(([p.numpy() for p in pinned], rs))
        h2d += sum(len(s) for s in seeds) * 4 + (len(seeds) + 1) * 8 + 16 * len(seeds)
    host_losses = [torch.empty(len(staged[k][0]), dtype=torch.float64).pin_memory() for k in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, (order, losses) in enumerate(pipe.run_windows(staged)):
        # per-batch losses of every step copied back to pinned host memory
        # (asynchronous D2H on the caller's stream; no per-step host stall)
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


def allreduce_probe(pipe, torch, world, device):
    """NVLink all-reduce of this job's gradient bucket (latency) and of a
    64 MiB buffer (bus bandwidth), CUDA events, max over ranks."""
    import torch.distributed as dist

    from paper_2409_14939_b200 import dist as fdist
    out = {"backend": str(dist.get_backend())}
    for name, numel in (("bucket", pipe.model.grad.numel()), ("64MiB", 16 << 20)):
        buf = torch.ones(numel, dtype=torch.float32, device=device)
        for _ in range(5):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50 if name == "bucket" else 10
        e0.record()
        for _ in range(reps):
            dist.all_reduce(buf)
        e1.record()
        torch.cuda.synchronize()
        t = fdist.max_over_ranks(e0.elapsed_time(e1) / reps / 1e3, world, device)
        nbytes = numel * 4
        out[name] = {"bytes": nbytes, "us": t * 1e6, "busbw_gbs": 2 * (world - 1) / world * nbytes / t / 1e9}
    return out


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
    _CPU.update(g=g, feats=_host_features(feats, cfg), labels=labels.cpu().numpy(), dims=cfg["dims"],
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
        "config": dict(config_dict(cfg, args, world, nbatches), host_processes=cores),
        "epoch_time_s": None,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
