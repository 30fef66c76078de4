"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from the unmodified reference).  CPU only."""

import hashlib

import numpy as np
import pytest

import oracle
from oracle import philox
from helpers import golden_graph, golden_layers


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_philox_stream_matches_numpy(golden):
    st = golden("philox")
    for i, s in enumerate(st["seeds"]):
        key = philox.key_for_seed(int(s))
        assert np.array_equal(np.array(key, dtype=np.uint64), st[f"key{i}"])
        u = st[f"u{i}"]
        assert np.array_equal(philox.uniform(key, 0, len(u)), u)
        # arbitrary absolute positions (unaligned starts)
        for start in (1, 2, 3, 5, 997):
            assert np.array_equal(philox.uniform(key, start, 4), u[start : start + 4])


def test_derive_seed(golden):
    st = golden("philox")
    want = st["derive"]
    got = [oracle.derive_seed(0, 13, j) for j in range(8)] + [
        oracle.derive_seed(3, 7), oracle.derive_seed(3, 11), oracle.derive_seed(3, 101)]
    assert np.array_equal(np.array(got, dtype=np.uint64), want)


def test_generator_digests(golden_meta, powerlaw_10k, cfg1_graph):
    d = golden_meta["graph_digest"]
    g = powerlaw_10k
    assert digest(g.row_offsets, g.col_indices, g.t_row_offsets, g.t_col_indices) == d["powerlaw_10k_16_7"]
    g = cfg1_graph
    assert g.num_edges == d["powerlaw_100k_10_1_edges"]
    assert digest(g.row_offsets, g.col_indices, g.t_row_offsets, g.t_col_indices) == d["powerlaw_100k_10_1"]


def test_sampler_cases(golden, golden_meta, powerlaw_10k):
    st = golden("sampler")
    for ci, case in enumerate(golden_meta["cases"]):
        g = powerlaw_10k if case["graph"] == "powerlaw_10k" else golden_graph(st, case["graph"])
        b = oracle.sample_khop(g, st[f"c{ci}_seeds"], case["fanouts"], int(case["seed"]))
        want = golden_layers(st, f"c{ci}", case["hops"])
        assert len(b.layers) == len(want)
        for (t, s, w), (t2, s2, w2) in zip(b.layers, want):
            assert np.array_equal(t, t2) and t.dtype == t2.dtype
            assert np.array_equal(s, s2) and s.dtype == s2.dtype
            assert np.array_equal(w, w2) and w.dtype == w2.dtype
        assert np.array_equal(b.unique_nodes, st[f"c{ci}_uniq"])


def test_sampler_cfg1_digests(golden_meta, cfg1_graph):
    tr, _ = oracle.train_split(cfg1_graph.num_nodes, 0)
    batches = oracle.epoch_seed_batches(tr, 1024, oracle.derive_seed(0, 11))
    assert len(batches) == 79
    for rec in golden_meta["cfg1"]:
        j = rec["batch"]
        b = oracle.sample_khop(cfg1_graph, batches[j], [10, 5], oracle.derive_seed(0, 13, j))
        assert digest(b.seeds) == rec["seeds_digest"]
        assert [len(t) for t, _, _ in b.layers] == rec["edges"]
        assert digest(*[a for lay in b.layers for a in lay]) == rec["layers_digest"]
        assert digest(b.unique_nodes) == rec["unique_digest"]


def test_idmap_traces(golden_meta):
    for tr in golden_meta["idmap_traces"]:
        t = oracle.idmap_build(tr["ids"], capacity_override=tr["cap"], hash_kind=tr["kind"])
        assert t.capacity == tr["capacity"] and t.shift == tr["shift"]
        assert [int(k) for k in t.keys] == tr["keys"]
        assert [int(v) for v in t.values] == tr["values"]
        assert t.num_inserted == tr["num_inserted"]


def test_idmap_layouts(golden):
    st = golden("idmap")
    for name in ("rand_u62", "dups", "sorted", "bench_ids"):
        t = oracle.idmap_build(st[f"{name}_ids"])
        assert np.array_equal(t.keys, st[f"{name}_keys"])
        assert np.array_equal(t.values, st[f"{name}_values"])
        got = oracle.idmap_lookup(t, st[f"{name}_ids"])
        occ = t.keys != oracle.SENTINEL
        assert len(np.unique(got)) == occ.sum()
    with pytest.raises(KeyError):
        oracle.idmap_lookup(oracle.idmap_build([1, 2, 3]), [4])


@pytest.mark.parametrize("arch", ["gcn", "gin"])
def test_prepare_forward_backward(golden, arch, powerlaw_10k):
    st = golden("compute")
    b = oracle.sample_khop(powerlaw_10k, st["seeds"], [6, 4], 77)
    local, seed_locals, n, csr = oracle.prepare_batch(b, arch)
    assert np.array_equal(seed_locals, st[f"{arch}_seed_locals"])
    for i, (lt, ls, _) in enumerate(local):
        assert np.array_equal(lt, st[f"{arch}_local_t{i}"])
        assert np.array_equal(ls, st[f"{arch}_local_s{i}"])
    for li, lay in enumerate(csr):
        for k, name in enumerate(("ip", "ix", "w", "tip", "tix", "tw")):
            assert np.array_equal(lay[k], st[f"{arch}_L{li}_{name}"]), (li, name)
    params = [[st[f"{arch}_W{i}"].copy(), st[f"{arch}_b{i}"].copy()] for i in range(2)]
    out, caches = oracle.forward(st[f"{arch}_x0"], csr, params, arch)
    for i, (_, h, z) in enumerate(caches):
        assert np.array_equal(h, st[f"{arch}_h{i}"])  # aggregation is bit-exact
        np.testing.assert_allclose(z, st[f"{arch}_z{i}"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(out, st[f"{arch}_out"], rtol=1e-5, atol=1e-6)
    loss, dl = oracle.softmax_xent(out[seed_locals], st[f"{arch}_labels"])
    assert loss == pytest.approx(float(st[f"{arch}_loss"][0]), rel=1e-6)
    dout = np.zeros_like(out)
    dout[seed_locals] = dl
    grads = oracle.backward(dout, caches, csr, params, arch)
    for i, (dw, db) in enumerate(grads):
        np.testing.assert_allclose(dw, st[f"{arch}_dW{i}"], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(db, st[f"{arch}_db{i}"], rtol=1e-5, atol=1e-6)


def test_aggregation_cases(golden):
    st = golden("compute")
    for c in range(3):
        ip, ix, w, x = (st[f"agg{c}_{k}"] for k in ("ip", "ix", "w", "x"))
        assert np.array_equal(oracle.aggregate(ip, ix, w, x), st[f"agg{c}_out"])
        tip, tix, tw = oracle.csr_transpose(ip, ix, w, len(x))
        assert np.array_equal(tip, st[f"agg{c}_tip"]) and np.array_equal(tix, st[f"agg{c}_tix"])
        assert np.array_equal(tw, st[f"agg{c}_tw"])
        assert np.array_equal(oracle.aggregate(tip, tix, tw, st[f"agg{c}_gy"]), st[f"agg{c}_bwd"])
    got = oracle.dense(st["dense_h"], st["dense_W"], st["dense_b"], relu=True)
    np.testing.assert_allclose(got, st["dense_relu"], rtol=1e-6, atol=1e-6)


def test_plan_tiles_table(golden_meta):
    for p in golden_meta["plan_tiles"]:
        err = oracle.tile_plan_error(p["nt"], p["d"], p["fanouts"], p["x"], p["y"], p["scratch"])
        assert (err is None) == (p["ok"] is True), p


def test_schedule_windows(golden, golden_meta):
    st = golden("schedule")
    for wi, rec in enumerate(golden_meta["schedule"]["windows"]):
        sets = [st[f"w{wi}_b{j}"] for j in range(6)]
        m = oracle.match_matrix(sets)
        assert np.array_equal(m, st[f"w{wi}_m"])
        order, ex, loads, traffic = oracle.window_schedule(sets, True, 32)
        assert order == rec["order"] and traffic == rec["traffic"]
        assert [len(x) for x in loads[1:]] == rec["loads"]
        assert oracle.window_schedule(sets, False, 32)[3] == rec["traffic_plain"]
    sets = [st[f"w0_b{j}"] for j in range(6)]
    order, ex, loads, _ = oracle.window_schedule(sets, True, 32)
    io = golden_meta["schedule"]["io"]
    for match in (True, False):
        got = oracle.epoch_h2d_bytes([ex], [loads], 32, match=match)
        assert list(got) == io[f"{match}_0.0"]


def test_static_cache_io(golden, golden_meta, powerlaw_10k):
    """Static-degree cache ratio 0.1 (memsim.py:110-186) on window 0 of the
    schedule fixture: host-link / Match / cache bytes equal the reference's."""
    st = golden("schedule")
    sets = [st[f"w0_b{j}"] for j in range(6)]
    _, ex, loads, _ = oracle.window_schedule(sets, True, 32)
    deg = np.diff(powerlaw_10k.row_offsets.astype(np.int64))
    mask = oracle.cache_mask(powerlaw_10k.num_nodes, 0.1, deg)
    assert mask.sum() == 1000
    io = golden_meta["schedule"]["io"]
    for match in (True, False):
        got = oracle.epoch_h2d_bytes([ex], [loads], 32, match=match, cached=mask)
        assert list(got) == io[f"{match}_0.1"]


@pytest.mark.parametrize("name", ["gcn", "gin", "gcn_noreorder", "gcn3"])
def test_train_trajectory(golden_meta, name):
    g, x, labels = oracle.two_cluster_task(200, 16, 0)
    kw = {
        "gcn": dict(layer_dims=(16, 32, 2), fanouts=[4, 4]),
        "gin": dict(layer_dims=(16, 8, 2), fanouts=[3, 2], arch="gin"),
        "gcn_noreorder": dict(layer_dims=(16, 32, 2), fanouts=[4, 4], reorder=False, match=False),
        "gcn3": dict(layer_dims=(16, 12, 8, 2), fanouts=[3, 3, 2], lr=0.1),
    }[name]
    kw = {"lr": 0.3, **kw}
    rep, _ = oracle.train(g, x, labels, batch_size=40, window_n=3, epochs=3, seed=0, **kw)
    want = golden_meta["train"][name]
    np.testing.assert_allclose([r["loss"] for r in rep], want["losses"], rtol=1e-5)
    assert [r["accuracy"] for r in rep] == want["accuracy"]
    assert [r["bytes_h2d"] for r in rep] == want["bytes_h2d"]
    assert [r["bytes_match"] for r in rep] == want["bytes_match"]


def test_random_walk_golden(golden, powerlaw_10k):
    """oracle.sample_random_walk == the reference's sample_random_walk
    (sampler.py:142-186) on the golden walk cases (incl. duplicate seeds)."""
    st = golden("walk")
    for c in range(int(st["ncases"])):
        b = oracle.sample_random_walk(powerlaw_10k, st[f"c{c}_seeds"], int(st[f"c{c}_len"]), int(st[f"c{c}_seed"]))
        t, s, w = b.layers[0]
        assert np.array_equal(t, st[f"c{c}_t"]) and np.array_equal(s, st[f"c{c}_s"])
        assert np.array_equal(w, st[f"c{c}_w"]) and np.array_equal(b.unique_nodes, st[f"c{c}_u"])


def test_sage_extension_restatement():
    """GraphSAGE-mean is an extension (the reference has none):
    its edge weights are 1/indeg in fp64 -> f32 and each layer adds the root
    term, i.e. h = mean_{u in N(v)} x_u + x_v before the dense transform."""
    lt = np.array([0, 0, 0, 1, 2, 2])
    ls = np.array([1, 2, 3, 0, 0, 3])
    w = oracle.layer_edge_weights("sage", lt, ls, 4)
    assert w.dtype == np.float32
    assert np.array_equal(w, np.array([1 / 3, 1 / 3, 1 / 3, 1, 0.5, 0.5], dtype=np.float32))
    ip, ix, cw, *_ = oracle.edges_to_csr(4, lt, ls, w) + (None,) * 0
    x = np.arange(8, dtype=np.float32).reshape(4, 2)
    h = oracle.aggregate(ip, ix, cw, x) + x
    want_row0 = (x[1] * np.float32(1 / 3) + x[2] * np.float32(1 / 3)) + x[3] * np.float32(1 / 3) + x[0]
    np.testing.assert_allclose(h[0], want_row0, rtol=1e-6)
