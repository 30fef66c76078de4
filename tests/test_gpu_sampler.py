"""GPU parity of the Fused-Map window sampler vs the oracle and the reference's
golden vectors (bit-exact: layers, unique_nodes, local IDs, Philox stream)."""

import hashlib

import numpy as np
import pytest

import oracle
from helpers import golden_graph, golden_layers

pytestmark = pytest.mark.gpu


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def assert_same_batch(got, want):
    assert len(got.layers) == len(want.layers)
    for h, ((t, s, w), (t2, s2, w2)) in enumerate(zip(got.layers, want.layers)):
        assert t.dtype == np.uint64 and s.dtype == np.uint64 and w.dtype == np.float32
        assert np.array_equal(t, t2), f"hop {h} targets"
        assert np.array_equal(s, s2), f"hop {h} sources"
        assert np.array_equal(w, w2), f"hop {h} weights"
    assert np.array_equal(got.unique_nodes, want.unique_nodes)


def test_philox_words_known_answer():
    import torch
    from paper_2409_14939_b200 import _lib
    from oracle import philox
    for seed in (0, 7, 2**63 + 11):
        key = philox.key_for_seed(seed)
        for start, count in ((0, 37), (3, 1001), (123456789, 64)):
            out = torch.empty(count, dtype=torch.int64, device="cuda")
            _lib.call("fgl_philox_words", key[0], key[1], start, count, out.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
            got = out.cpu().numpy().view(np.uint64)
            assert np.array_equal(got, philox.raw_words(key, start, count))


def test_golden_cases(golden, golden_meta, powerlaw_10k):
    from paper_2409_14939_b200 import sampler
    st = golden("sampler")
    for ci, case in enumerate(golden_meta["cases"]):
        g = powerlaw_10k if case["graph"] == "powerlaw_10k" else golden_graph(st, case["graph"])
        got = sampler.sample_khop(g, st[f"c{ci}_seeds"], case["fanouts"], int(case["seed"]))
        want = golden_layers(st, f"c{ci}", case["hops"])
        for h, ((t, s, w), (t2, s2, w2)) in enumerate(zip(got.layers, want)):
            assert np.array_equal(t, t2) and np.array_equal(s, s2) and np.array_equal(w, w2), (ci, h)
        assert np.array_equal(got.unique_nodes, st[f"c{ci}_uniq"]), ci


def test_cfg1_digests(golden_meta, cfg1_graph):
    from paper_2409_14939_b200 import sampler
    tr, _ = oracle.train_split(cfg1_graph.num_nodes, 0)
    batches = oracle.epoch_seed_batches(tr, 1024, oracle.derive_seed(0, 11))
    for rec in golden_meta["cfg1"]:
        j = rec["batch"]
        b = sampler.sample_khop(cfg1_graph, batches[j], [10, 5], oracle.derive_seed(0, 13, j))
        assert [len(t) for t, _, _ in b.layers] == rec["edges"]
        assert digest(*[a for lay in b.layers for a in lay]) == rec["layers_digest"]
        assert digest(b.unique_nodes) == rec["unique_digest"]


@pytest.mark.parametrize("fan", [[1], [3, 2], [15, 10, 5], [33, 2], [64], [100, 3], [200], [256, 1]])
def test_random_graphs_vs_oracle(powerlaw_10k, fan):
    from paper_2409_14939_b200 import sampler
    rng = np.random.default_rng(sum(fan))
    for trial in range(4):
        seeds = rng.integers(0, 10_000, size=int(rng.integers(1, 700))).astype(np.uint64)
        s = int(rng.integers(0, 2**63))
        assert_same_batch(sampler.sample_khop(powerlaw_10k, seeds, fan, s),
                          oracle.sample_khop(powerlaw_10k, seeds, fan, s))


def test_window_local_ids(cfg1_graph):
    """A window of 8 batches in one call: per-batch parity, local IDs = rank in
    unique_nodes (trainer path of idmap.build, trainer.py:167), seed locals."""
    from paper_2409_14939_b200 import sampler
    from paper_2409_14939_b200.graph import device_graph
    dg = device_graph(cfg1_graph)
    rng = np.random.default_rng(4)
    sizes = [1024, 1024, 500, 1, 1024, 77, 1024, 1000]
    seed_lists = [rng.integers(0, cfg1_graph.num_nodes, size=n) for n in sizes]
    rng_seeds = [oracle.derive_seed(0, 13, j) for j in range(8)]
    ws = sampler.WindowSampler(dg, [10, 5], 1024, 8)
    win = ws.sample(seed_lists, rng_seeds)
    for b in range(8):
        got = win.to_batch(b)
        want = oracle.sample_khop(cfg1_graph, seed_lists[b], [10, 5], rng_seeds[b])
        assert_same_batch(got, want)
        assert win.draws(b) == want.draws
        for (lt, ls, _), (t, s, _) in zip(got.local_layers, want.layers):
            assert np.array_equal(lt, np.searchsorted(want.unique_nodes, t))
            assert np.array_equal(ls, np.searchsorted(want.unique_nodes, s))
        s0, s1 = int(win.seed_off_host[b]), int(win.seed_off_host[b + 1])
        u0 = win.unique_range(b)[0]
        seeds_b = seed_lists[b].astype(np.uint64)
        assert np.array_equal(ws.seed_rows[s0:s1].cpu().numpy() - u0,
                              np.searchsorted(want.unique_nodes, seeds_b))
        # block layout: frontier lists and frontier-indexed edges
        fronts = [np.unique(seeds_b)] + [np.unique(s) for _, s, _ in want.layers]
        for h in range(2):
            f0, f1 = win.front_range(h, b)
            fl = ws.frontier[h * ws.fcap + f0 : h * ws.fcap + f1].cpu().numpy().astype(np.uint64)
            assert np.array_equal(fl, fronts[h])
            e0, e1 = win.edge_range(h, b)
            t, s, _ = want.layers[h]
            assert np.array_equal(ws.tgt_front[e0:e1].cpu().numpy() - f0, np.searchsorted(fronts[h], t))
            sf = ws.src_front[e0:e1].cpu().numpy()
            if h == 0:
                g0 = win.front_range(1, b)[0]
                assert np.array_equal(sf - g0, np.searchsorted(fronts[1], s))
            else:
                assert np.array_equal(sf - u0, np.searchsorted(want.unique_nodes, s))
        f0 = win.front_range(0, b)[0]
        assert np.array_equal(ws.seed_front[s0:s1].cpu().numpy() - f0,
                              np.searchsorted(fronts[0], seeds_b))
    # the same sampler object is reusable for a smaller window
    win2 = ws.sample(seed_lists[:2], rng_seeds[:2])
    assert_same_batch(win2.to_batch(1), oracle.sample_khop(cfg1_graph, seed_lists[1], [10, 5], rng_seeds[1]))


def test_weighted_and_sink_graphs(golden):
    from paper_2409_14939_b200 import sampler
    st = golden("sampler")
    g = golden_graph(st, "weighted300")
    rng = np.random.default_rng(9)
    for _ in range(5):
        seeds = rng.integers(0, 300, size=20).astype(np.uint64)
        s = int(rng.integers(0, 2**62))
        assert_same_batch(sampler.sample_khop(g, seeds, [7, 5, 3], s), oracle.sample_khop(g, seeds, [7, 5, 3], s))
    path = golden_graph(st, "path4")
    assert_same_batch(sampler.sample_khop(path, [3], [2, 2], 4), oracle.sample_khop(path, [3], [2, 2], 4))


def test_validation_errors(powerlaw_10k):
    from paper_2409_14939_b200 import sampler
    from paper_2409_14939_b200.errors import ConfigError, ValidationError
    with pytest.raises(ValidationError):
        sampler.sample_khop(powerlaw_10k, [], [2], 0)
    with pytest.raises(ValidationError):
        sampler.sample_khop(powerlaw_10k, [10_000], [2], 0)
    with pytest.raises(ValidationError):
        sampler.sample_khop(powerlaw_10k, [1], [0], 0)
    with pytest.raises(ConfigError):
        sampler.sample_khop(powerlaw_10k, [1], [257], 0)


def test_streaming_select_path_parity():
    """The streaming top-list select kernel (FGL_SELECT=stream, used for
    fanouts > 128 and as the overflow fallback) is bit-exact too."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, oracle
from paper_2409_14939_b200 import sampler
g = oracle.gen_power_law(3000, 20, 2)
rng = np.random.default_rng(3)
for fan in ([5, 3], [15, 10, 5], [40, 2], [100]):
    seeds = rng.integers(0, 3000, size=300).astype(np.uint64)
    a = sampler.sample_khop(g, seeds, fan, 99)
    b = oracle.sample_khop(g, seeds, fan, 99)
    for (t, s, w), (t2, s2, w2) in zip(a.layers, b.layers):
        assert np.array_equal(t, t2) and np.array_equal(s, s2)
    assert np.array_equal(a.unique_nodes, b.unique_nodes)
print("ok")
'''
    env = dict(os.environ, FGL_SELECT="stream")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
