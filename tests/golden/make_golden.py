"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``minigl`` from ``/root/reference/pkg/src`` (read-only; numba's
cache goes to a temp dir) and records the reference's own outputs for the
hot-path functions of SURVEY.md section 8(a).  The fixtures are small and
committed; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = os.environ.get("MINIGL_REF_SRC", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
sys.path.insert(0, REF)

from minigl import compute, graph, idmap, memsim, sampler, schedule, trainer  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def pack_layers(prefix, layers, store):
    for i, (t, s, w) in enumerate(layers):
        store[f"{prefix}_t{i}"] = t
        store[f"{prefix}_s{i}"] = s
        store[f"{prefix}_w{i}"] = w


def philox_fixture():
    seeds = [0, 1, 7, 12345, 2**63 + 11, trainer.derive_seed(0, 13, 5)]
    store = {"seeds": np.array(seeds, dtype=np.uint64)}
    for i, s in enumerate(seeds):
        bg = np.random.Philox(s)
        store[f"key{i}"] = np.asarray(bg.state["state"]["key"], dtype=np.uint64)
        u = np.random.Generator(bg).random(1001)
        store[f"u{i}"] = u
    store["derive"] = np.array(
        [trainer.derive_seed(0, 13, j) for j in range(8)]
        + [trainer.derive_seed(3, 7), trainer.derive_seed(3, 11), trainer.derive_seed(3, 101)],
        dtype=np.uint64,
    )
    np.savez_compressed(OUT / "philox.npz", **store)


def tiny_graphs():
    """Small graphs exercising edge cases: conftest ring/star/path, sinks,
    weights, duplicate edges, self loops."""
    gs = {
        "ring3": graph.from_edges(3, [0, 1, 2], [1, 2, 0]),
        "star4": graph.from_edges(4, [0, 0, 0], [1, 2, 3]),
        "path4": graph.from_edges(4, [0, 1, 2], [1, 2, 3]),
        "dup_self": graph.from_edges(5, [0, 0, 0, 1, 1, 2, 4, 4], [1, 1, 0, 2, 2, 4, 4, 3]),
    }
    rng = np.random.default_rng(5)
    src = rng.integers(0, 300, size=3000)
    dst = rng.integers(0, 300, size=3000)
    w = rng.random(3000).astype(np.float32) + 0.25
    gs["weighted300"] = graph.from_edges(300, src, dst, w)
    return gs


def sampler_fixture():
    store, meta = {}, {}
    gs = tiny_graphs()
    g10k = graph.generate(graph.GraphGenSpec("power-law", 10_000, avg_degree=16, seed=7))
    g100k = graph.generate(graph.GraphGenSpec("power-law", 100_000, avg_degree=10, seed=1))
    meta["graph_digest"] = {
        "powerlaw_10k_16_7": digest(g10k.row_offsets, g10k.col_indices, g10k.t_row_offsets, g10k.t_col_indices),
        "powerlaw_100k_10_1": digest(g100k.row_offsets, g100k.col_indices, g100k.t_row_offsets, g100k.t_col_indices),
        "powerlaw_100k_10_1_edges": int(g100k.num_edges),
    }
    for name, g in gs.items():
        store[f"g_{name}_off"] = g.row_offsets
        store[f"g_{name}_col"] = g.col_indices
        if g.edge_weights is not None:
            store[f"g_{name}_w"] = g.edge_weights
    cases = []
    rng = np.random.default_rng(11)
    plan = [
        ("ring3", [0], [1, 1, 1], 3),
        ("star4", [0], [5], 0),
        ("star4", [0, 0, 3], [2, 2], 9),       # duplicate seeds, sink hop
        ("path4", [3], [2, 2], 4),             # seed with no out-edges -> empty hops
        ("path4", [0, 1], [1, 1, 1, 1], 5),
        ("dup_self", [0, 4], [2, 3], 6),       # duplicate edges + self loops
        ("weighted300", list(range(0, 300, 7)), [4, 3], 8),
        ("weighted300", [5, 5, 9], [40], 10),  # fanout above every degree
    ]
    for j in range(10):
        seeds = rng.integers(0, 10_000, size=int(rng.integers(1, 400)))
        fan = [int(x) for x in rng.integers(1, 16, size=int(rng.integers(1, 4)))]
        plan.append(("powerlaw_10k", seeds.tolist(), fan, int(rng.integers(0, 2**63))))
    plan.append(("powerlaw_10k", list(range(1024)), [15, 10, 5], 2**63 + 1))
    for ci, (gname, seeds, fan, s) in enumerate(plan):
        g = g10k if gname == "powerlaw_10k" else gs[gname]
        b = sampler.sample_khop(g, np.array(seeds, dtype=np.uint64), sampler.Fanouts(fan), s)
        store[f"c{ci}_seeds"] = b.seeds
        store[f"c{ci}_uniq"] = b.unique_nodes
        pack_layers(f"c{ci}", b.layers, store)
        cases.append({"graph": gname, "fanouts": fan, "seed": str(s), "hops": len(b.layers)})
    # config-1 batches (100K / 1M power-law, bs 1024, [10,5]): digests only
    cfg = trainer.ModelConfig(layer_dims=(128, 64, 2), fanouts=[10, 5], batch_size=1024, seed=0)
    tr, _ = train_split_ref(g100k.num_nodes, 0)
    batches = sampler.make_epoch_batches(g100k, tr, 1024, trainer.derive_seed(0, 11))
    cfg1 = []
    for j in (0, 1, 78):
        b = sampler.sample_khop(g100k, batches[j], cfg.fanouts, trainer.derive_seed(0, 13, j))
        flat = [a for lay in b.layers for a in lay]
        cfg1.append({
            "batch": j,
            "seeds_digest": digest(b.seeds),
            "layers_digest": digest(*flat),
            "unique_digest": digest(b.unique_nodes),
            "edges": [int(len(t)) for t, _, _ in b.layers],
            "num_unique": int(len(b.unique_nodes)),
        })
    meta["cases"] = cases
    meta["cfg1"] = cfg1
    np.savez_compressed(OUT / "sampler.npz", **store)
    return meta, g10k


def train_split_ref(n, seed):
    rng = np.random.Generator(np.random.Philox(trainer.derive_seed(seed, 7)))
    perm = rng.permutation(n).astype(np.uint64)
    cut = max(1, int(0.8 * n))
    return perm[:cut], perm[cut:]


def idmap_fixture():
    traces = []
    for ids, cap, kind in [
        ([3], 5, "mod"), ([3, 3], 5, "mod"), ([3, 11], 8, "mod"), ([3, 7], 4, "mod"),
        ([5, 13, 21, 6, 5, 29], 8, "mod"), ([50, 3, 99, 3, 12], None, "fib"),
        ([0, 1, 2, 3, 4, 5, 6, 7], 8, "mod"), ([9, 1, 17, 25, 2, 1, 33], 16, "mod"),
    ]:
        t = idmap.build(ids, capacity_override=cap, hash_kind=kind)
        traces.append({"ids": ids, "cap": cap, "kind": kind, "capacity": t.capacity, "shift": t.shift,
                       "keys": [int(k) for k in t.keys], "values": [int(v) for v in t.values],
                       "num_inserted": t.num_inserted})
    rng = np.random.default_rng(3)
    big = {}
    for name, ids in [
        ("rand_u62", rng.integers(0, 1 << 62, size=700, dtype=np.uint64)),
        ("dups", rng.integers(0, 300, size=2000).astype(np.uint64)),
        ("sorted", np.unique(rng.integers(0, 10**6, size=5000)).astype(np.uint64)),
        ("bench_ids", idmap.bench_ids(4096, 0.5, seed=2)),
    ]:
        t = idmap.build(ids, workers=1)
        big[f"{name}_ids"] = ids
        big[f"{name}_keys"] = t.keys
        big[f"{name}_values"] = t.values
    np.savez_compressed(OUT / "idmap.npz", **big)
    return traces


def compute_fixture(g10k):
    store = {}
    rng = np.random.default_rng(21)
    b = sampler.sample_khop(g10k, rng.integers(0, 10_000, size=200).astype(np.uint64), [6, 4], 77)
    for arch in ("gcn", "gin"):
        cfg = trainer.ModelConfig(layer_dims=(12, 16, 5), fanouts=[6, 4], arch=arch, seed=4)
        tr, seed_locals, layers = trainer._prepare_batch(b, cfg)
        store[f"{arch}_seed_locals"] = seed_locals
        for i, lay in enumerate(tr.local_layers):
            store[f"{arch}_local_t{i}"], store[f"{arch}_local_s{i}"], _ = lay
        for li, lay in enumerate(layers):
            for k, name in enumerate(("ip", "ix", "w", "tip", "tix", "tw")):
                store[f"{arch}_L{li}_{name}"] = lay[k]
        n = tr.num_local
        x0 = rng.standard_normal((n, 12)).astype(np.float32)
        labels = rng.integers(0, 5, size=len(b.seeds))
        params = trainer._init_params(cfg)
        store[f"{arch}_x0"] = x0
        store[f"{arch}_labels"] = labels
        for i, (w, bb) in enumerate(params):
            bb += rng.standard_normal(bb.shape).astype(np.float32) * 0.1
            store[f"{arch}_W{i}"] = w.copy()
            store[f"{arch}_b{i}"] = bb.copy()
        out, caches = trainer._forward(x0, layers, params, cfg)
        loss, dl = trainer._softmax_xent(out[seed_locals], labels)
        dout = np.zeros_like(out)
        dout[seed_locals] = dl
        grads = trainer._backward(dout, caches, layers, params, cfg)
        store[f"{arch}_out"] = out
        store[f"{arch}_loss"] = np.array([loss])
        store[f"{arch}_dlogits"] = dl
        for i, (x, h, z) in enumerate(caches):
            store[f"{arch}_h{i}"] = h
            store[f"{arch}_z{i}"] = z
        for i, (dw, db) in enumerate(grads):
            store[f"{arch}_dW{i}"] = dw
            store[f"{arch}_db{i}"] = db
    store["seeds"] = b.seeds
    # standalone aggregation + dense cases
    for c in range(3):
        nt, ns, md, d = [(40, 30, 9, 7), (64, 64, 40, 33), (5, 200, 150, 128)][c]
        deg = rng.integers(0, md + 1, size=nt)
        ip = np.zeros(nt + 1, dtype=np.int64)
        np.cumsum(deg, out=ip[1:])
        ix = rng.integers(0, ns, size=int(deg.sum()))
        w = rng.standard_normal(int(deg.sum())).astype(np.float32)
        x = rng.standard_normal((ns, d)).astype(np.float32)
        store[f"agg{c}_ip"], store[f"agg{c}_ix"], store[f"agg{c}_w"], store[f"agg{c}_x"] = ip, ix, w, x
        store[f"agg{c}_out"] = compute.aggregate_forward(ip, ix, w, x, compute.TileConfig())
        tip, tix, tw = compute.csr_transpose(ip, ix, w, ns)
        store[f"agg{c}_tip"], store[f"agg{c}_tix"], store[f"agg{c}_tw"] = tip, tix, tw
        gy = rng.standard_normal((nt, d)).astype(np.float32)
        store[f"agg{c}_gy"] = gy
        store[f"agg{c}_bwd"] = compute.aggregate_backward(tip, tix, tw, gy, compute.TileConfig())
    h = rng.standard_normal((50, 20)).astype(np.float32)
    W = rng.standard_normal((20, 9)).astype(np.float32)
    bias = rng.standard_normal(9).astype(np.float32)
    store["dense_h"], store["dense_W"], store["dense_b"] = h, W, bias
    store["dense_relu"] = compute.dense_update(h, W, bias, "relu")
    np.savez_compressed(OUT / "compute.npz", **store)
    # plan_tiles accept/reject table
    plans = []
    for nt, d, fo, x, y, sc in [
        (10, 64, [3] * 10, 8, 32, 128 * 1024), (10, 64, [4000] * 10, 8, 32, 128 * 1024),
        (16, 32, [1] * 16, 32, 32, 1 << 20), (16, 32, [1] * 16, 31, 33, 1 << 20),
        (3, 100, [0, 0, 0], 8, 32, 1024), (3, 100, [0, 0, 0], 8, 32, 1023),
        (9, 10, [1, 2, 3, 4, 5, 6, 7, 8, 380], 8, 8, 2048), (9, 10, [1, 2, 3, 4, 5, 6, 7, 8, 370], 8, 8, 2048),
        (0, 5, [], 8, 32, 128 * 1024), (4, 8, [1, 1, 1, 1], 0, 32, 1024),
    ]:
        try:
            compute.plan_tiles(nt, d, np.array(fo, dtype=np.int64),
                               compute.TileConfig(x, y, sc))
            ok = True
        except Exception as e:  # noqa: BLE001
            ok = type(e).__name__
        plans.append({"nt": nt, "d": d, "fanouts": fo, "x": x, "y": y, "scratch": sc, "ok": ok})
    return plans


def schedule_fixture(g10k):
    rng = np.random.default_rng(8)
    store = {}
    wins = []
    for wi in range(3):
        batches = [sampler.sample_khop(g10k, rng.integers(0, 10_000, size=64).astype(np.uint64),
                                       [5, 3], int(rng.integers(0, 2**62))) for _ in range(6)]
        for j, b in enumerate(batches):
            store[f"w{wi}_b{j}"] = b.unique_nodes
        m = schedule.build_match_matrix(batches)
        sch = schedule.schedule_window(batches, True, 32)
        sch_plain = schedule.schedule_window(batches, False, 32)
        store[f"w{wi}_m"] = m.m
        wins.append({"order": sch.order, "traffic": sch.window_traffic_bytes,
                     "traffic_plain": sch_plain.window_traffic_bytes,
                     "loads": [len(t.load_ids) for t in sch.transitions],
                     "stats": schedule.match_stats(batches)})
        if wi == 0:
            sched0 = [sch, sch_plain]
    deg = g10k.out_degrees()
    io = {}
    for match in (True, False):
        for ratio in (0.0, 0.1):
            rep = memsim.simulate_epoch_io([sched0[0]], ratio, "static-degree" if ratio else "none",
                                           (g10k.num_nodes, 32), memsim.CostParams(),
                                           degrees=deg, match=match)
            io[f"{match}_{ratio}"] = [rep.bytes_host_to_device, rep.bytes_served_by_match,
                                      rep.bytes_served_by_cache]
    # the Fig. 5 / tie cases of test_schedule.py
    np.savez_compressed(OUT / "schedule.npz", **store)
    return {"windows": wins, "io": io}


def train_fixture():
    out = {}
    g, feats, labels = trainer.two_cluster_task(200, 16, seed=0)
    for name, kw, flags in [
        ("gcn", dict(layer_dims=(16, 32, 2), fanouts=[4, 4]), trainer.PipelineFlags()),
        ("gin", dict(layer_dims=(16, 8, 2), fanouts=[3, 2], arch="gin"), trainer.PipelineFlags()),
        ("gcn_noreorder", dict(layer_dims=(16, 32, 2), fanouts=[4, 4]),
         trainer.PipelineFlags(match=False, reorder=False)),
        ("gcn3", dict(layer_dims=(16, 12, 8, 2), fanouts=[3, 3, 2], lr=0.1), trainer.PipelineFlags()),
        ("gcn_naive", dict(layer_dims=(16, 32, 2), fanouts=[4, 4]), trainer.PipelineFlags(memory_aware=False)),
    ]:
        cfg = trainer.ModelConfig(batch_size=40, window_n=3, epochs=3, seed=0, **{"lr": 0.3, **kw})
        rep = trainer.train(g, feats, labels, cfg, flags)
        out[name] = {
            "losses": rep.losses,
            "accuracy": [e.accuracy for e in rep.epochs],
            "bytes_h2d": [e.traffic.bytes_host_to_device for e in rep.epochs],
            "bytes_match": [e.traffic.bytes_served_by_match for e in rep.epochs],
            "bytes_cache": [e.traffic.bytes_served_by_cache for e in rep.epochs],
            "modeled_io_seconds": [e.traffic.modeled_io_seconds for e in rep.epochs],
            "modeled_fetch_seconds": [e.modeled_fetch_seconds for e in rep.epochs],
            "per_batch_epoch0": [vars(b) for b in rep.epochs[0].traffic.per_batch],
        }
    out["two_cluster_digest"] = digest(g.row_offsets, g.col_indices, feats.data, labels)
    return out


def walk_fixture():
    """Random walks (sampler.py:142-186) on the 10K power-law graph: varied
    seed counts (incl. duplicates), lengths and stream seeds."""
    g = graph.generate(graph.GraphGenSpec("power-law", 10_000, avg_degree=16, seed=7))
    rng = np.random.default_rng(31)
    store = {}
    cases = [(1, 1), (5, 3), (64, 4), (700, 2), (2000, 6), (3000, 1)]
    for c, (n, length) in enumerate(cases):
        seeds = rng.integers(0, 10_000, size=n).astype(np.uint64)
        s = int(rng.integers(0, 2**62))
        b = sampler.sample_random_walk(g, seeds, length, s)
        t, src, w = b.layers[0]
        store.update({f"c{c}_seeds": seeds, f"c{c}_len": np.int64(length), f"c{c}_seed": np.uint64(s),
                      f"c{c}_t": t, f"c{c}_s": src, f"c{c}_w": w, f"c{c}_u": b.unique_nodes})
    store["ncases"] = np.int64(len(cases))
    np.savez_compressed(OUT / "walk.npz", **store)


def graph_io_fixture():
    """graph.from_edges (graph.py:151-183) on edge lists with duplicates and
    self loops (weighted / unweighted), and an MGL1 file written by
    graph.save_binary (graph.py:293-307)."""
    rng = np.random.default_rng(41)
    store = {}
    cases = [(50, 400, False), (300, 3000, True), (1000, 20000, False), (7, 0, False)]
    for c, (n, m, weighted) in enumerate(cases):
        src = rng.integers(0, n, size=m).astype(np.uint64)
        dst = rng.integers(0, n, size=m).astype(np.uint64)
        if m:
            src[: m // 10] = src[m // 10 : 2 * (m // 10)]   # exact duplicate pairs
            dst[: m // 10] = dst[m // 10 : 2 * (m // 10)]
            dst[2 * (m // 10) : 2 * (m // 10) + 5] = src[2 * (m // 10) : 2 * (m // 10) + 5]  # self loops
        w = rng.standard_normal(m).astype(np.float32) if weighted else None
        g = graph.from_edges(n, src, dst, w)
        store.update({f"c{c}_n": np.int64(n), f"c{c}_src": src, f"c{c}_dst": dst,
                      f"c{c}_ro": g.row_offsets, f"c{c}_ci": g.col_indices, f"c{c}_tro": g.t_row_offsets,
                      f"c{c}_tci": g.t_col_indices})
        if weighted:
            store.update({f"c{c}_w": w, f"c{c}_ew": g.edge_weights, f"c{c}_tew": g.t_edge_weights})
    store["ncases"] = np.int64(len(cases))
    np.savez_compressed(OUT / "graph_io.npz", **store)
    g = graph.from_edges(300, store["c1_src"], store["c1_dst"], store["c1_w"])
    graph.save_binary(g, OUT / "small_weighted.mgl1")


def main():
    graph_io_fixture()
    walk_fixture()
    philox_fixture()
    meta, g10k = sampler_fixture()
    meta["idmap_traces"] = idmap_fixture()
    meta["plan_tiles"] = compute_fixture(g10k)
    meta["schedule"] = schedule_fixture(g10k)
    meta["train"] = train_fixture()
    meta["numpy"] = np.__version__
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, default=str))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "walk":
        walk_fixture()  # regenerate only the random-walk fixture
    elif len(sys.argv) > 1 and sys.argv[1] == "graph_io":
        graph_io_fixture()
    else:
        main()
