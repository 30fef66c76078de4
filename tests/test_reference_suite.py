"""The reference package's own test suite, restated against the drop-in
modules (SURVEY 8(c) "rerunning the reference's own tests"; VERDICT r1
missing #6).  The reference's tests cannot run on the GPU box (its source
does not travel there), so every hot-path test class of
/root/reference/pkg/tests is restated here, case for case, with the same
inputs, oracles and tolerances, calling this package's sampler / idmap /
compute / schedule / trainer / memsim.  Each test names the reference test it
restates (file:line).  Tests that only exercise host logic (plan_tiles,
make_epoch_batches, the memsim formulas) run without a GPU; the rest are
marked gpu.  Out of scope: test_cli.py, the text
edge-list parser and generators of test_graph.py, memsim.simulate_epoch_io
(replaced by the loader's measured counts, tests/test_gpu_cache.py)."""

from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from paper_2409_14939_b200 import compute, graph, idmap, memsim, sampler, schedule, trainer
from paper_2409_14939_b200.compute import TileConfig
from paper_2409_14939_b200.errors import ConfigError, NotFoundError, ValidationError
from paper_2409_14939_b200.sampler import Fanouts, SubgraphBatch

gpu = pytest.mark.gpu


# ----------------------------------------------------------------- fixtures --
# (reference conftest.py:8-37)
def _star4():
    return graph.from_edges(4, [0, 0, 0], [1, 2, 3])


def _path4():
    return graph.from_edges(4, [0, 1, 2], [1, 2, 3])


@pytest.fixture(scope="module")
def pl10k():
    """graph.generate(power-law, 10_000, avg_degree 16, seed 7), restated by
    the oracle generator (pinned to the reference in test_oracle_golden)."""
    return oracle.gen_power_law(10_000, 16, 7)


def _ids_batch(ids):
    ids = np.unique(np.asarray(ids, dtype=np.uint64))
    e = np.empty(0, dtype=np.uint64)
    return SubgraphBatch(seeds=ids[:1], layers=[(e, e, np.empty(0, np.float32))], unique_nodes=ids)


def _fw_edges(g):
    off = np.asarray(g.row_offsets, dtype=np.int64)
    col = np.asarray(g.col_indices, dtype=np.int64)
    return {(u, int(col[e])) for u in range(g.num_nodes) for e in range(off[u], off[u + 1])}


def _rand_csr(rng, nt, ns, max_deg, dim):
    deg = rng.integers(0, max_deg + 1, size=nt)
    ip = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(deg, out=ip[1:])
    ix = rng.integers(0, ns, size=int(deg.sum()))
    w = rng.standard_normal(int(deg.sum())).astype(np.float32)
    x = rng.standard_normal((ns, dim)).astype(np.float32)
    return ip, ix, w, x


def _dense64(ip, ix, w, x):
    a = np.zeros((len(ip) - 1, len(x)), dtype=np.float64)
    for t in range(len(ip) - 1):
        for e in range(ip[t], ip[t + 1]):
            a[t, ix[e]] += w[e]
    return a @ x.astype(np.float64)


# ------------------------------------------------------- test_compute.py --
@gpu
class TestComputeForward:
    def test_single_edge_identity(self):  # test_compute.py:32-36
        ip, ix, w = compute.edges_to_csr(1, [0], [0], [1.0])
        x = np.array([[3.0, -2.0, 5.0]], dtype=np.float32)
        assert np.array_equal(compute.aggregate_forward(ip, ix, w, x, TileConfig()), x)

    def test_convex_combination(self):  # :38-42
        ip, ix, w = compute.edges_to_csr(1, [0, 0], [0, 1], [0.5, 0.5])
        x = np.array([[2.0, 4.0], [2.0, 4.0]], dtype=np.float32)
        assert np.allclose(compute.aggregate_forward(ip, ix, w, x, TileConfig()), [[2.0, 4.0]])

    def test_zero_fanout_rows_exactly_zero(self):  # :44-51
        ip = np.array([0, 0, 1, 1], dtype=np.int64)
        x = np.full((2, 3), 7.0, dtype=np.float32)
        out = compute.aggregate_forward(ip, np.array([0]), np.ones(1, np.float32), x, TileConfig())
        assert np.all(out[0] == 0.0) and np.all(out[2] == 0.0) and np.array_equal(out[1], x[0])

    @pytest.mark.parametrize("seed", range(6))
    def test_matches_dense_oracle(self, seed):  # :53-59
        ip, ix, w, x = _rand_csr(np.random.default_rng(seed), 50, 50, 12, 64)
        assert np.allclose(compute.aggregate_forward(ip, ix, w, x, TileConfig()), _dense64(ip, ix, w, x),
                           rtol=1e-5, atol=1e-5)

    def test_tiling_invariance(self):  # :61-66
        ip, ix, w, x = _rand_csr(np.random.default_rng(11), 37, 37, 9, 21)
        outs = [compute.aggregate_forward(ip, ix, w, x, c) for c in (TileConfig(8, 32), TileConfig(4, 16),
                                                                      TileConfig(1, 1))]
        for o in outs[1:]:
            assert np.allclose(outs[0], o, rtol=1e-6, atol=0.0)

    def test_oversized_tile_rejected_before_compute(self):  # :68-72
        ip, ix, w, x = _rand_csr(np.random.default_rng(0), 8, 8, 3, 4)
        with pytest.raises(ConfigError):
            compute.aggregate_forward(ip, ix, w, x, TileConfig(16, 64))

    def test_budget_violation_rejected_before_compute(self):  # :74-79
        ip, ix, w = compute.edges_to_csr(1, [0] * 30, list(range(30)), [1.0] * 30)
        with pytest.raises(ConfigError, match="reduce targets_per_tile"):
            compute.aggregate_forward(ip, ix, w, np.ones((30, 4), np.float32),
                                      TileConfig(8, 32, scratch_limit_bytes=1100))


@gpu
class TestComputeBackward:
    def test_chain_rule_single_edge(self):  # test_compute.py:83-91
        ip, ix, w = compute.edges_to_csr(2, [0], [1], [0.75])
        t = compute.csr_transpose(ip, ix, w, 2)
        g = compute.aggregate_backward(*t, np.ones((2, 3), np.float32), TileConfig())
        assert np.allclose(g[1], 0.75) and np.all(g[0] == 0.0)

    def test_zero_grad_out(self):  # :93-97
        ip, ix, w = compute.edges_to_csr(3, [0, 1], [1, 2], [1.0, 2.0])
        t = compute.csr_transpose(ip, ix, w, 3)
        assert np.all(compute.aggregate_backward(*t, np.zeros((3, 4), np.float32), TileConfig()) == 0.0)

    @pytest.mark.parametrize("seed", range(4))
    def test_finite_differences(self, seed):  # :99-120
        rng = np.random.default_rng(100 + seed)
        ip, ix, w, x = _rand_csr(rng, 10, 10, 4, 6)
        probe = rng.standard_normal((10, 6)).astype(np.float32)
        grad = compute.aggregate_backward(*compute.csr_transpose(ip, ix, w, 10), probe, TileConfig())
        eps, p64 = 1e-3, probe.astype(np.float64)
        fd = np.zeros(x.shape)
        for i in range(x.shape[0]):
            for j in range(x.shape[1]):
                xp, xm = x.astype(np.float64), x.astype(np.float64)
                xp[i, j] += eps
                xm[i, j] -= eps
                fd[i, j] = ((_dense64(ip, ix, w, xp) * p64).sum() - (_dense64(ip, ix, w, xm) * p64).sum()) / (2 * eps)
        assert np.allclose(grad, fd, rtol=1e-4, atol=1e-4 * max(1.0, np.abs(fd).max()))

    @pytest.mark.parametrize("seed", range(4))
    def test_adjoint_identity(self, seed):  # :122-131
        rng = np.random.default_rng(200 + seed)
        ip, ix, w, x = _rand_csr(rng, 20, 20, 6, 8)
        probe = rng.standard_normal((20, 8)).astype(np.float32)
        fwd = compute.aggregate_forward(ip, ix, w, x, TileConfig())
        bwd = compute.aggregate_backward(*compute.csr_transpose(ip, ix, w, 20), probe, TileConfig())
        lhs = float((fwd.astype(np.float64) * probe).sum())
        rhs = float((bwd.astype(np.float64) * x).sum())
        assert lhs == pytest.approx(rhs, rel=1e-5, abs=1e-5)


class TestPlanTiles:  # test_compute.py:134-172 (host logic)
    def test_default_single_tile(self):
        assert compute.plan_tiles(8, 32, np.full(8, 3), TileConfig(8, 32)).num_tiles == 1

    def test_ceiling_arithmetic(self):
        assert compute.plan_tiles(9, 33, np.full(9, 3), TileConfig(8, 32)).num_tiles == 4

    def test_scratch_budget_value(self):
        plan = compute.plan_tiles(8, 32, np.full(8, 15), TileConfig(8, 32))
        assert plan.row_groups[0][3] == 4 * 8 * 32 + 4 * 8 * 15 == 1504

    def test_thread_cap_rejected(self):
        for cfg in (TileConfig(16, 64), TileConfig(33, 32)):
            with pytest.raises(ConfigError):
                compute.plan_tiles(4, 4, np.zeros(4), cfg)

    def test_single_heavy_target_suggests_smaller_tile(self):
        with pytest.raises(ConfigError, match="reduce targets_per_tile"):
            compute.plan_tiles(1, 4, np.array([100000]), TileConfig(8, 32, scratch_limit_bytes=2048))

    def test_tiles_cover_each_cell_once(self):
        seen = np.zeros((11, 13), dtype=int)
        for t0, t1, c0, c1 in compute.plan_tiles(11, 13, np.zeros(11), TileConfig(4, 5)).tiles:
            seen[t0:t1, c0:c1] += 1
        assert np.all(seen == 1)

    def test_fanout_length_validated(self):
        with pytest.raises(ValidationError):
            compute.plan_tiles(3, 4, np.zeros(2), TileConfig())


@gpu
class TestDenseUpdate:  # test_compute.py:175-207
    def test_identity(self):
        h = np.arange(6, dtype=np.float32).reshape(2, 3)
        assert np.array_equal(compute.dense_update(h, np.eye(3, dtype=np.float32)), h)

    def test_relu_clamps(self):
        out = compute.dense_update(np.array([[1.0, -1.0]], np.float32), -np.eye(2, dtype=np.float32),
                                   activation="relu")
        assert out.tolist() == [[0.0, 1.0]]

    def test_triple_loop_oracle(self):
        rng = np.random.default_rng(4)
        h = rng.standard_normal((10, 8)).astype(np.float32)
        w = rng.standard_normal((8, 4)).astype(np.float32)
        b = rng.standard_normal(4).astype(np.float32)
        expect = h.astype(np.float64) @ w.astype(np.float64) + b.astype(np.float64)
        assert np.allclose(compute.dense_update(h, w, b), expect, rtol=1e-6, atol=1e-6)

    def test_dim_mismatch(self):
        with pytest.raises(ValidationError):
            compute.dense_update(np.ones((2, 3), np.float32), np.ones((4, 2), np.float32))


# ------------------------------------------------------- test_sampler.py --
@gpu
class TestKhop:
    def test_star_fanout_above_degree_takes_all(self):  # test_sampler.py:18-23
        t, s, w = sampler.sample_khop(_star4(), [0], Fanouts([5]), seed=0).layers[0]
        assert sorted(s.tolist()) == [1, 2, 3] and t.tolist() == [0, 0, 0] and np.all(w == 1.0)

    def test_two_layer_fanout_two_edge_bound(self, pl10k):  # :25-29
        b = sampler.sample_khop(pl10k, [0], Fanouts([2, 2]), seed=1)
        assert len(b.layers[0][0]) <= 2 and len(b.layers[1][0]) <= 4 and b.num_sampled_edges() <= 6

    def test_deterministic(self):  # :31-38
        g = graph.from_edges(100, np.arange(100), (np.arange(100) + 1) % 100)
        seeds = np.arange(10, dtype=np.uint64)
        b1 = sampler.sample_khop(g, seeds, Fanouts([1, 1]), seed=3)
        b2 = sampler.sample_khop(g, seeds, Fanouts([1, 1]), seed=3)
        assert np.array_equal(b1.unique_nodes, b2.unique_nodes)
        for l1, l2 in zip(b1.layers, b2.layers):
            assert all(np.array_equal(a, b) for a, b in zip(l1, l2))

    def test_empty_and_out_of_range_seeds_rejected(self):  # :40-46
        for seeds in ([], [9]):
            with pytest.raises(ValidationError):
                sampler.sample_khop(_star4(), seeds, Fanouts([2]), seed=0)

    def test_weights_carried(self):  # :48-51
        g = graph.from_edges(2, [0], [1], [2.5])
        assert sampler.sample_khop(g, [0], Fanouts([3]), seed=0).layers[0][2].tolist() == [2.5]

    def test_layer_targets_come_from_previous_frontier(self, pl10k):  # :53-57
        b = sampler.sample_khop(pl10k, [1, 2, 3], Fanouts([3, 3]), seed=9)
        assert set(b.layers[0][0].tolist()) <= {1, 2, 3}
        assert set(b.layers[1][0].tolist()) <= set(b.layers[0][1].tolist())


@gpu
class TestRandomWalk:  # test_sampler.py:60-90
    def test_isolated_seed(self):
        b = sampler.sample_random_walk(graph.from_edges(2, [1], [0]), [0], length=3, seed=0)
        assert b.unique_nodes.tolist() == [0] and b.num_sampled_edges() == 0

    def test_forced_path_walk(self):
        t, s, _ = sampler.sample_random_walk(_path4(), [0], length=3, seed=5).layers[0]
        assert list(zip(t.tolist(), s.tolist())) == [(0, 1), (1, 2), (2, 3)]

    def test_walk_unique_bound(self, pl10k):
        b = sampler.sample_random_walk(pl10k, np.arange(1000, dtype=np.uint64), length=3, seed=2)
        assert b.num_unique <= 4000

    def test_length_validated(self):
        with pytest.raises(ValidationError):
            sampler.sample_random_walk(_path4(), [0], length=0, seed=0)

    def test_deterministic(self, pl10k):
        a = sampler.sample_random_walk(pl10k, [5, 6], length=4, seed=11)
        b = sampler.sample_random_walk(pl10k, [5, 6], length=4, seed=11)
        assert np.array_equal(a.layers[0][1], b.layers[0][1])


class TestEpochBatches:  # test_sampler.py:93-118 (host logic)
    def test_sizes_and_single_batch(self, pl10k):
        assert [len(b) for b in sampler.make_epoch_batches(pl10k, np.arange(10), 4, shuffle_seed=0)] == [4, 4, 2]
        big = sampler.make_epoch_batches(pl10k, np.arange(10), 64, shuffle_seed=0)
        assert len(big) == 1 and len(big[0]) == 10

    def test_deterministic_partition(self, pl10k):
        a = sampler.make_epoch_batches(pl10k, np.arange(100), 7, shuffle_seed=9)
        b = sampler.make_epoch_batches(pl10k, np.arange(100), 7, shuffle_seed=9)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))

    def test_is_partition(self, pl10k):
        ids = np.arange(53, dtype=np.uint64)
        joined = np.sort(np.concatenate(sampler.make_epoch_batches(pl10k, ids, 8, shuffle_seed=1)))
        assert np.array_equal(joined, ids)

    def test_batch_size_validated(self, pl10k):
        with pytest.raises(ValidationError):
            sampler.make_epoch_batches(pl10k, np.arange(4), 0, shuffle_seed=0)


_graph_cases = st.integers(3, 14).flatmap(lambda n: st.tuples(
    st.just(n), st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1)), max_size=50),
    st.lists(st.integers(0, n - 1), min_size=1, max_size=4), st.lists(st.integers(1, 4), min_size=1, max_size=3),
    st.integers(0, 2**31)))


@gpu
class TestKhopProperties:  # test_sampler.py:121-153
    @given(_graph_cases)
    @settings(max_examples=60, deadline=None)
    def test_sampled_edges_subset_counts_and_unique_set(self, case):
        n, edges, seeds, fanouts, seed = case
        g = graph.from_edges(n, [u for u, _ in edges], [v for _, v in edges])
        b = sampler.sample_khop(g, np.array(seeds, np.uint64), Fanouts(fanouts), seed)
        gset = _fw_edges(g)
        deg = np.diff(np.asarray(g.row_offsets, np.int64))
        frontier = np.unique(np.array(seeds, np.uint64))
        seen = set(seeds)
        for (t, s, _), f in zip(b.layers, fanouts):
            assert all((int(u), int(v)) in gset for u, v in zip(t, s))
            cnt = dict(zip(*np.unique(t, return_counts=True))) if len(t) else {}
            for u in frontier.tolist():
                assert cnt.get(u, 0) == min(int(deg[u]), f)
            frontier = np.unique(s)
            seen |= set(t.tolist()) | set(s.tolist())
        assert b.unique_nodes.tolist() == sorted(seen)


# --------------------------------------------------------- test_idmap.py --
SENT = int(idmap.SENTINEL)


def _assert_bijection(table, ids):  # test_idmap.py:12-22
    occ = table.keys != idmap.SENTINEL
    expect = np.unique(np.asarray(ids, np.uint64))
    assert np.array_equal(np.sort(table.keys[occ]), expect)
    assert np.array_equal(np.sort(table.values[occ]), np.arange(len(expect), dtype=np.uint64))
    assert table.num_inserted == len(expect)


@gpu
class TestIdMap:
    def test_traces(self):  # test_idmap.py:25-54
        t = idmap.build([3], capacity_override=5, hash_kind="mod")
        assert t.keys[3] == 3 and t.values[3] == 0 and t.num_inserted == 1
        t = idmap.build([3, 3], capacity_override=5, hash_kind="mod")
        assert t.num_inserted == 1 and np.count_nonzero(t.keys != idmap.SENTINEL) == 1
        t = idmap.build([3, 11], capacity_override=8, hash_kind="mod")
        assert (t.keys[3], t.values[3], t.keys[4], t.values[4]) == (3, 0, 11, 1)
        t = idmap.build([3, 7], capacity_override=4, hash_kind="mod")
        assert t.keys[3] == 3 and t.keys[0] == 7

    def test_rejections(self):  # :56-62
        for ids in ([SENT], []):
            with pytest.raises(ValidationError):
                idmap.build(ids)

    def test_single_thread_first_seen_order_and_capacity(self):  # :64-73
        t = idmap.build([50, 3, 99, 3, 12], workers=1)
        assert [idmap.lookup(t, g) for g in (50, 3, 99, 12)] == [0, 1, 2, 3]
        t = idmap.build(np.arange(1000, dtype=np.uint64))
        assert t.capacity >= 2000 and t.capacity & (t.capacity - 1) == 0

    def test_lookup(self):  # :76-94
        assert idmap.lookup(idmap.build([3], capacity_override=5, hash_kind="mod"), 3) == 0
        with pytest.raises(NotFoundError, match="7"):
            idmap.lookup(idmap.build([3]), 7)
        ids = np.random.default_rng(0).integers(0, 1 << 60, size=10_000, dtype=np.uint64)
        t = idmap.build(ids, workers=4)
        _assert_bijection(t, ids)
        locs = idmap.lookup_many(t, np.unique(ids))
        assert np.array_equal(np.sort(locs), np.arange(t.num_inserted, dtype=np.uint64))

    def test_translate(self):  # :114-163
        b = SubgraphBatch(seeds=np.array([3], np.uint64),
                          layers=[(np.array([3, 7], np.uint64), np.array([7, 3], np.uint64), np.ones(2, np.float32))],
                          unique_nodes=np.array([3, 7], np.uint64))
        out = idmap.translate_batch(idmap.build([3, 7], workers=1), b)
        lt, ls, _ = out.local_layers[0]
        assert list(zip(lt.tolist(), ls.tolist())) == [(0, 1), (1, 0)] and out.num_local == 2
        rng = np.random.default_rng(3)
        nodes = rng.choice(1 << 40, size=50, replace=False).astype(np.uint64)
        ti, si = rng.integers(0, 50, 200), rng.integers(0, 50, 200)
        b = SubgraphBatch(seeds=nodes[:5], layers=[(nodes[ti], nodes[si], np.ones(200, np.float32))],
                          unique_nodes=np.unique(nodes))
        table = idmap.build(b.unique_nodes)
        lt, ls, _ = idmap.translate_batch(table, b).local_layers[0]
        inv = np.empty(table.num_inserted, dtype=np.uint64)
        occ = table.keys != idmap.SENTINEL
        inv[table.values[occ].astype(np.int64)] = table.keys[occ]
        assert np.array_equal(inv[lt], nodes[ti]) and np.array_equal(inv[ls], nodes[si])
        b = SubgraphBatch(seeds=np.array([1], np.uint64),
                          layers=[(np.array([1], np.uint64), np.array([42], np.uint64), np.ones(1, np.float32))],
                          unique_nodes=np.array([1, 42], np.uint64))
        with pytest.raises(NotFoundError, match="42"):
            idmap.translate_batch(idmap.build([1]), b)

    @pytest.mark.parametrize("ids,cap", [([3], 5), ([3, 3], 5), ([3, 11], 8)])
    def test_locked_baseline_matches_build(self, ids, cap):  # :166-183
        a = idmap.build(ids, capacity_override=cap, hash_kind="mod")
        b = idmap.build_locked_baseline(ids, capacity_override=cap, hash_kind="mod")
        assert np.array_equal(a.keys, b.keys) and np.array_equal(a.values, b.values)

    def test_bench_helpers(self):  # :208-219
        ids = idmap.bench_ids(10_000, 0.9, seed=1)
        assert len(ids) == 10_000 and len(np.unique(ids)) == 1_000
        r = idmap.run_bench(20_000, workers=2, dup_ratio=0.5, seed=0, repeats=1)
        assert r["n_unique"] == 10_000 and r["build_ns"] > 0 and r["baseline_ns"] > 0
        assert r["speedup"] == pytest.approx(r["baseline_ns"] / r["build_ns"])

    @given(st.lists(st.integers(0, 2**50), min_size=1, max_size=300), st.sampled_from([1, 2, 3, 4]))
    @settings(max_examples=40, deadline=None)
    def test_bijection_any_schedule(self, ids, workers):  # :187-193
        _assert_bijection(idmap.build(np.array(ids, np.uint64), workers=workers), ids)

    @given(st.lists(st.integers(0, 2**40), min_size=2, max_size=100, unique=True))
    @settings(max_examples=30, deadline=None)
    def test_lookup_injective(self, ids):  # :202-206
        locs = idmap.lookup_many(idmap.build(np.array(ids, np.uint64), workers=2), np.array(ids, np.uint64))
        assert len(set(locs.tolist())) == len(ids)


# ------------------------------------------------------ test_schedule.py --
def _straight_greedy(m):  # test_schedule.py:11-31: literal row / column zeroing
    m = np.array(m, dtype=float)
    n = len(m)
    np.fill_diagonal(m, 0.0)
    order, used, z = [0], {0}, 0
    for _ in range(n - 1):
        best, h = 0.0, None
        for k in range(n):
            if k not in used and m[z][k] > best:
                best, h = m[z][k], k
        h = min(set(range(n)) - used) if h is None else h
        order.append(h)
        used.add(h)
        m[z, :] = 0.0
        m[:, z] = 0.0
        z = h
    return order


@gpu
class TestSchedule:
    def test_match_degree(self):  # test_schedule.py:35-50
        assert schedule.match_degree([1, 2, 3], [1, 2, 3]) == 1.0
        assert schedule.match_degree([1, 2], [3, 4]) == 0.0
        assert schedule.match_degree([0, 3, 4, 10, 12], [0, 3, 4, 7, 9]) == pytest.approx(0.6)
        with pytest.raises(ValidationError):
            schedule.match_degree([], [1])

    @given(st.lists(st.integers(0, 30), min_size=1, max_size=20), st.lists(st.integers(0, 30), min_size=1, max_size=20))
    @settings(max_examples=40, deadline=None)
    def test_match_degree_brute_force(self, a, b):  # :52-59
        sa, sb = set(a), set(b)
        assert schedule.match_degree(a, b) == pytest.approx(len(sa & sb) / min(len(sa), len(sb)))

    def test_match_matrix(self):  # :62-84
        m = schedule.build_match_matrix([_ids_batch([1, 2]), _ids_batch([1, 2])]).m
        assert m[0, 1] == m[1, 0] == 1.0 and m[0, 0] == m[1, 1] == 0.0
        assert np.all(schedule.build_match_matrix([_ids_batch([10 * i, 10 * i + 1]) for i in range(4)]).m == 0.0)
        rng = np.random.default_rng(0)
        m = schedule.build_match_matrix([_ids_batch(rng.integers(0, 40, size=12)) for _ in range(5)]).m
        assert np.array_equal(m, m.T)
        with pytest.raises(ValidationError):
            schedule.build_match_matrix([_ids_batch([1])])

    def test_greedy_cases(self):  # :87-107
        m = np.array([[0.0, 0.2, 0.6], [0.2, 0.0, 0.3], [0.6, 0.3, 0.0]])
        assert schedule.greedy_reorder(schedule.MatchMatrix(3, m)) == [0, 2, 1]
        assert schedule.greedy_reorder(schedule.MatchMatrix(4, np.zeros((4, 4)))) == [0, 1, 2, 3]
        m = np.zeros((3, 3))
        m[0, 1] = m[0, 2] = m[1, 2] = m[2, 1] = 0.5
        assert schedule.greedy_reorder(schedule.MatchMatrix(3, m)) == [0, 1, 2]

    @given(st.integers(0, 10_000))
    @settings(max_examples=60, deadline=None)
    def test_greedy_matches_straight_line_trace(self, seed):  # :109-118
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 8))
        m = rng.random((n, n))
        m = (m + m.T) / 2
        np.fill_diagonal(m, 0.0)
        assert schedule.greedy_reorder(schedule.MatchMatrix(n, m)) == _straight_greedy(m)

    def test_transitions(self):  # :134-150
        ov, ld = schedule.compute_transition(_ids_batch([0, 3, 4, 7, 9]), _ids_batch([0, 3, 4, 10, 12]))
        assert ov.tolist() == [0, 3, 4] and ld.tolist() == [10, 12]
        b = _ids_batch([1, 5, 9])
        assert schedule.compute_transition(b, b)[1].size == 0
        ov, ld = schedule.compute_transition(_ids_batch([1]), _ids_batch([2, 3]))
        assert ov.size == 0 and ld.tolist() == [2, 3]

    @given(st.lists(st.lists(st.integers(0, 25), min_size=1, max_size=15), min_size=2, max_size=6))
    @settings(max_examples=40, deadline=None)
    def test_transition_partition_property(self, windows):  # :152-162
        sched = schedule.schedule_window([_ids_batch(ids) for ids in windows], enable_reorder=True, feature_dim=4)
        for j, tr in enumerate(sched.transitions):
            assert np.array_equal(np.union1d(tr.overlap_ids, tr.load_ids), sched.batch_nodes[j + 1])
            assert np.intersect1d(tr.overlap_ids, tr.load_ids).size == 0

    def test_schedule_window(self):  # :165-196
        b = _ids_batch([1, 2, 3])
        s = schedule.schedule_window([b], enable_reorder=True, feature_dim=8)
        assert s.window_traffic_bytes == 3 * 8 * 4 and s.transitions == []
        s = schedule.schedule_window([b, b], enable_reorder=False, feature_dim=8)
        assert len(s.transitions[0].load_ids) == 0 and s.window_traffic_bytes == 3 * 8 * 4
        bs = [_ids_batch([0, 3, 4, 7, 9]), _ids_batch([0, 5, 6, 8, 11]), _ids_batch([0, 3, 4, 10, 12])]
        on, off = schedule.schedule_window(bs, True, feature_dim=2), schedule.schedule_window(bs, False, feature_dim=2)
        assert on.order == [0, 2, 1] and on.window_traffic_bytes <= off.window_traffic_bytes
        st_ = schedule.match_stats([_ids_batch([0, 1, 2]), _ids_batch([1, 2, 3]), _ids_batch([9])])
        assert 0.0 <= st_["avg_match_degree"] <= 1.0 and st_["delta_match"] >= 0.0


# ------------------------------------------------------- test_trainer.py --
def _cfg(**kw):  # test_trainer.py:15-26
    base = dict(layer_dims=(16, 32, 2), fanouts=Fanouts([4, 4]), batch_size=40, window_n=3, epochs=6, lr=0.3, seed=0)
    base.update(kw)
    return trainer.ModelConfig(**base)


@pytest.fixture(scope="module")
def task():
    return oracle.two_cluster_task(200, 16, 0)


@gpu
class TestTrain:
    def test_loss_halves_on_two_clusters(self, task):  # test_trainer.py:30-35
        losses = trainer.train(*task, _cfg(epochs=10)).losses
        assert losses[-1] <= 0.5 * losses[0] and all(np.isfinite(losses))

    def test_zero_lr_keeps_loss_flat(self, task):  # :37-41
        losses = np.array(trainer.train(*task, _cfg(lr=0.0, epochs=4)).losses)
        assert np.allclose(losses, losses[0], rtol=1e-12, atol=1e-12)

    def test_accounting_flags_leave_trajectory_unchanged(self, task):  # :43-53
        off = trainer.PipelineFlags(match=False, reorder=False, memory_aware=False)
        on = trainer.PipelineFlags(match=True, reorder=False, memory_aware=True)
        r_off, r_on = trainer.train(*task, _cfg(epochs=5), off), trainer.train(*task, _cfg(epochs=5), on)
        for a, b in zip(r_off.losses, r_on.losses):
            assert a == pytest.approx(b, abs=1e-4)
        assert r_on.epochs[0].traffic.bytes_served_by_match >= 0
        assert r_off.epochs[0].traffic.bytes_served_by_match == 0

    def test_same_seed_reproduces_trajectory(self, task):  # :55-60
        a, b = trainer.train(*task, _cfg(epochs=3)), trainer.train(*task, _cfg(epochs=3))
        assert a.losses == b.losses and [e.accuracy for e in a.epochs] == [e.accuracy for e in b.epochs]

    def test_reorder_still_trains(self, task):  # :62-66
        r = trainer.train(*task, _cfg(epochs=8), trainer.PipelineFlags(reorder=True))
        assert r.losses[-1] <= 0.6 * r.losses[0]

    def test_validation_before_epoch_zero(self, task):  # :68-73
        g, x, y = task
        with pytest.raises(ValidationError):
            trainer.train(g, x, y, _cfg(layer_dims=(8, 4, 2)))
        with pytest.raises(ValidationError):
            trainer.train(g, x, y[:100], _cfg())

    def test_gin_trains(self, task):  # :75-78
        r = trainer.train(*task, _cfg(arch="gin", epochs=8, lr=0.05))
        assert r.losses[-1] < r.losses[0]

    def test_traffic_matches_match_flag(self, task):  # :80-84
        on = trainer.train(*task, _cfg(epochs=1), trainer.PipelineFlags(match=True, reorder=False))
        off = trainer.train(*task, _cfg(epochs=1), trainer.PipelineFlags(match=False, reorder=False))
        assert on.epochs[0].traffic.bytes_host_to_device <= off.epochs[0].traffic.bytes_host_to_device

    def test_memory_aware_lowers_modeled_fetch(self, task):  # :86-90
        aware = trainer.train(*task, _cfg(epochs=1), trainer.PipelineFlags(memory_aware=True))
        naive = trainer.train(*task, _cfg(epochs=1), trainer.PipelineFlags(memory_aware=False))
        assert aware.epochs[0].modeled_fetch_seconds < naive.epochs[0].modeled_fetch_seconds


@gpu
class TestPhaseBreakdown:  # test_trainer.py:112-141
    def test_percentages_sum_to_100(self, task):
        pct = trainer.phase_breakdown(trainer.train(*task, _cfg(epochs=2)))
        assert set(pct) == set(trainer.PHASES) and sum(pct.values()) == pytest.approx(100.0, abs=0.1)

    def test_empty_report_rejected(self):
        with pytest.raises(ValidationError):
            trainer.phase_breakdown(trainer.TrainReport(config=_cfg(), flags=trainer.PipelineFlags()))


# -------------------------------------------------------- test_memsim.py --
def _fetch_oracle(f, d, sbw, gbw):  # test_memsim.py:14-22 (exact rationals)
    naive = Fraction(4 * (f - 1) * d + 8 * f * d) / Fraction(gbw)
    aware = Fraction(4 * (f - 1) * d + 4 * f * (d - 1)) / Fraction(sbw) + Fraction(4 * f * d + 4 * f) / Fraction(gbw)
    return float(naive), float(aware)


class TestFetchTimes:  # test_memsim.py:25-73 (host formulas)
    def test_unit_bandwidth_and_reference_values(self):
        assert memsim.t_naive(1, 1, memsim.CostParams(shared_bw=8, global_bw=4, host_link_bw=1)) == pytest.approx(2.0)
        p = memsim.CostParams()
        naive, aware = _fetch_oracle(10, 256, 12_000_000_000_000, 938_000_000_000)
        assert memsim.t_naive(10, 256, p) == pytest.approx(naive, rel=1e-12)
        assert memsim.t_memory_aware(10, 256, p) == pytest.approx(aware, rel=1e-12)
        assert naive == pytest.approx(29696 / 938e9, rel=1e-12)

    def test_naive_linear_and_equal_bandwidths(self):
        p = memsim.CostParams()
        for f in (1, 5, 16):
            for d in (1, 7, 128):
                assert memsim.t_naive(f, 2 * d, p) == pytest.approx(2 * memsim.t_naive(f, d, p), rel=1e-12)
        p = memsim.CostParams(shared_bw=1e9, global_bw=1e9)
        assert memsim.t_memory_aware(9, 33, p) == pytest.approx(memsim.t_naive(9, 33, p), rel=1e-12)

    @given(st.integers(1, 64), st.integers(1, 1024), st.floats(1e9, 1e13), st.floats(1.01, 100.0))
    @settings(max_examples=200, deadline=None)
    def test_memory_aware_never_slower(self, f, d, gbw, ratio):
        p = memsim.CostParams(shared_bw=gbw * ratio, global_bw=gbw)
        aware, naive = memsim.t_memory_aware(f, d, p), memsim.t_naive(f, d, p)
        assert aware <= naive * (1 + 1e-12)
        if (f, d) != (1, 1):
            assert aware < naive

    def test_validation(self):
        p = memsim.CostParams()
        for call in (lambda: memsim.t_naive(0, 4, p), lambda: memsim.t_memory_aware(4, 0, p),
                     lambda: memsim.t_naive(4, 4, memsim.CostParams(global_bw=0))):
            with pytest.raises(ValidationError):
                call()
