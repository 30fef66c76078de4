"""GPU parity of the full training step (prepare -> SpMM -> dense -> loss ->
backward -> SGD) against the oracle and the reference's golden trajectories.
Tolerances: aggregation bit-exact; dense/loss/grads 1e-5 relative (north star)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _task():
    return oracle.two_cluster_task(200, 16, 0)


_TRAJ = {
    "gcn": (dict(layer_dims=(16, 32, 2), fanouts=[4, 4]), {}),
    "gin": (dict(layer_dims=(16, 8, 2), fanouts=[3, 2], arch="gin"), {}),
    "gcn_noreorder": (dict(layer_dims=(16, 32, 2), fanouts=[4, 4]), dict(match=False, reorder=False)),
    "gcn3": (dict(layer_dims=(16, 12, 8, 2), fanouts=[3, 3, 2], lr=0.1), {}),
    "gcn_naive": (dict(layer_dims=(16, 32, 2), fanouts=[4, 4]), dict(memory_aware=False)),
}


@pytest.mark.parametrize("name", sorted(_TRAJ))
def test_train_matches_reference_trajectory(golden_meta, name):
    """trainer.train end to end against the reference's own 3-epoch run:
    accuracies, IO bytes (totals and per batch), modeled IO / fetch seconds
    exact; epoch-mean losses after 3 free-running epochs within 2e-4 (the
    per-step 1e-5 bar is test_trajectory_per_step_1e5 below)."""
    from paper_2409_14939_b200 import trainer
    g, x, labels = _task()
    kw = _TRAJ[name]
    cfg = trainer.ModelConfig(batch_size=40, window_n=3, epochs=3, seed=0, **{"lr": 0.3, **kw[0]})
    rep = trainer.train(g, x, labels, cfg, trainer.PipelineFlags(**kw[1]))
    want = golden_meta["train"][name]
    np.testing.assert_allclose(rep.losses, want["losses"], rtol=2e-4, atol=1e-6)
    assert [e.traffic.bytes_host_to_device for e in rep.epochs] == want["bytes_h2d"]
    assert [e.traffic.bytes_served_by_match for e in rep.epochs] == want["bytes_match"]
    assert [e.traffic.bytes_served_by_cache for e in rep.epochs] == want["bytes_cache"]
    assert [e.traffic.modeled_io_seconds for e in rep.epochs] == want["modeled_io_seconds"]
    assert [e.modeled_fetch_seconds for e in rep.epochs] == want["modeled_fetch_seconds"]
    assert [vars(b) for b in rep.epochs[0].traffic.per_batch] == want["per_batch_epoch0"]
    assert rep.epochs[0].traffic.to_dict()["per_batch"] == want["per_batch_epoch0"]
    assert [e.accuracy for e in rep.epochs] == want["accuracy"]


@pytest.mark.parametrize("name", ["gcn", "gin", "gcn3", "gcn_noreorder"])
def test_trajectory_per_step_1e5(name):
    """The 3-epoch trajectory of the golden configs, checked per window at the
    north-star 1e-5: before every window the oracle takes the GPU's current
    parameters, replays the window's batches in the GPU's schedule order
    (sample_khop, prepare, forward, fp64 loss, backward, SGD), and every
    per-batch loss and the parameters after the window must agree within
    1e-5 relative -- so fp32 rounding differences cannot accumulate."""
    from paper_2409_14939_b200 import trainer
    from paper_2409_14939_b200.sampler import make_epoch_batches
    g, x, labels = _task()
    kw = _TRAJ[name]
    cfg = trainer.ModelConfig(batch_size=40, window_n=3, epochs=3, seed=0, **{"lr": 0.3, **kw[0]})
    flags = trainer.PipelineFlags(**kw[1])
    feats = x.data if hasattr(x, "data") else x
    pipe = trainer.Pipeline(g, x, labels, cfg, flags)
    perm = np.random.Generator(np.random.Philox(oracle.derive_seed(0, 7))).permutation(g.num_nodes)
    train_ids = perm[: max(1, int(0.8 * g.num_nodes))].astype(np.uint64)
    batches = make_epoch_batches(g, train_ids, cfg.batch_size, oracle.derive_seed(0, 11))
    windows = [batches[i : i + cfg.window_n] for i in range(0, len(batches), cfg.window_n)]
    steps = 0
    for _ in range(cfg.epochs):
        base = 0
        for ws in windows:
            rs = [oracle.derive_seed(0, 13, base + j) for j in range(len(ws))]
            base += len(ws)
            params = pipe.model.to_numpy()
            order, losses = pipe.run_window([w.astype(np.int64) for w in ws], rs)
            lv = losses.cpu().numpy()
            ob = [oracle.sample_khop(g, w, cfg.fanouts, r) for w, r in zip(ws, rs)]
            o_order = oracle.window_schedule([b.unique_nodes for b in ob], flags.reorder, cfg.layer_dims[0])[0]
            assert order == o_order
            for j, bi in enumerate(order):
                loss, _ = oracle.train_step(ob[bi], feats, labels, params, cfg.lr, cfg.arch)
                assert lv[j] / len(ws[bi]) == pytest.approx(loss, rel=1e-5)
                steps += 1
            for (w, b), (w2, b2) in zip(pipe.model.to_numpy(), params):
                np.testing.assert_allclose(w, w2, rtol=1e-5, atol=1e-5 * float(np.abs(w2).max()))
                np.testing.assert_allclose(b, b2, rtol=1e-5, atol=1e-5 * max(float(np.abs(b2).max()), 1e-3))
    assert steps == cfg.epochs * len(batches)


@pytest.mark.parametrize("arch,dims,fan,direct", [("gcn", (128, 64, 2), [10, 5], False),
                                                  ("gcn", (128, 64, 2), [10, 5], True),
                                                  ("gcn", (128, 48, 32, 7), [6, 4, 3], True),
                                                  ("gcn", (32, 64, 172), [6, 4], True),  # papers' classes: fused top, CW 192
                                                  ("gin", (128, 16, 3), [5, 3], False)])
def test_window_steps_match_oracle(cfg1_graph, arch, dims, fan, direct):
    """A window of 4 batches on config 1: per-batch loss and the parameters
    after every SGD step track the oracle within 1e-5 relative."""
    import torch
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(1)
    feats = rng.standard_normal((g.num_nodes, dims[0])).astype(np.float32)
    labels = rng.integers(0, dims[-1], size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=dims, fanouts=fan, arch=arch, batch_size=512, window_n=4,
                              lr=0.1, seed=3)
    pipe = trainer.Pipeline(g, feats, labels, cfg, trainer.PipelineFlags(reorder=True), direct_x0=direct)
    params = oracle.init_params(dims, 3)
    seeds = [rng.choice(g.num_nodes, 512, replace=False) for _ in range(4)]
    rs = [oracle.derive_seed(3, 13, j) for j in range(4)]
    order, losses = pipe.run_window(seeds, rs)
    batches = [oracle.sample_khop(g, s, fan, r) for s, r in zip(seeds, rs)]
    o_order, ex, _, _ = oracle.window_schedule([b.unique_nodes for b in batches], True, dims[0])
    assert order == o_order
    lv = losses.cpu().numpy()
    for j, bi in enumerate(o_order):
        loss, _ = oracle.train_step(batches[bi], feats, labels, params, cfg.lr, arch)
        assert lv[j] / len(seeds[bi]) == pytest.approx(loss, rel=1e-5)
    got = pipe.model.to_numpy()
    # 1e-5 relative to the parameter scale after 4 SGD steps: fp32 dense
    # products and partial sums round differently from numpy's BLAS
    for (w, b), (w2, b2) in zip(got, params):
        np.testing.assert_allclose(w, w2, rtol=1e-5, atol=1e-5 * float(np.abs(w2).max()))
        np.testing.assert_allclose(b, b2, rtol=1e-5, atol=1e-5 * max(float(np.abs(b2).max()), 0.1))
    torch.cuda.synchronize()


def test_io_accounting_matches_simulate_epoch_io(cfg1_graph):
    """Rows read from the feature store == memsim.simulate_epoch_io load sets."""
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(2)
    feats = rng.standard_normal((g.num_nodes, 12)).astype(np.float32)
    labels = rng.integers(0, 2, size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=(12, 8, 2), fanouts=[10, 5], batch_size=256, window_n=8,
                              lr=0.1, seed=0)
    pipe = trainer.Pipeline(g, feats, labels, cfg)
    seeds = [rng.choice(g.num_nodes, 256, replace=False) for _ in range(8)]
    rs = [oracle.derive_seed(0, 13, j) for j in range(8)]
    pipe.loaded.zero_()
    pipe.run_window(seeds, rs)
    batches = [oracle.sample_khop(g, s, [10, 5], r) for s, r in zip(seeds, rs)]
    _, ex, loads, traffic = oracle.window_schedule([b.unique_nodes for b in batches], True, 12)
    assert int(pipe.loaded.sum().item()) * 4 * 12 == traffic


def test_host_feature_store_bit_exact(cfg1_graph):
    """Pinned-host features (zero-copy delta loads) give the same training step."""
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(5)
    feats = rng.standard_normal((g.num_nodes, 20)).astype(np.float32)
    labels = rng.integers(0, 4, size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=(20, 16, 4), fanouts=[8, 4], batch_size=300, window_n=3, lr=0.2)
    seeds = [rng.choice(g.num_nodes, 300, replace=False) for _ in range(3)]
    rs = [11, 12, 13]
    out = []
    for store in ("device", "host"):
        pipe = trainer.Pipeline(g, feats, labels, cfg, feature_store=store)
        pipe.run_window(seeds, rs)
        out.append(pipe.model.flat.cpu().numpy())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("direct", [False, True])
def test_pipelined_windows_bit_identical(cfg1_graph, direct):
    """run_windows (window w+1 sampled on a side stream while window w trains)
    gives exactly the parameters and losses of run_window in sequence."""
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(9)
    feats = rng.standard_normal((g.num_nodes, 20)).astype(np.float32)
    labels = rng.integers(0, 4, size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=(20, 16, 16, 4), fanouts=[6, 4, 3], batch_size=200, window_n=4, lr=0.2)
    wins = [([rng.choice(g.num_nodes, 200, replace=False) for _ in range(4)], [100 * w + j for j in range(4)])
            for w in range(5)]
    seq = trainer.Pipeline(g, feats, labels, cfg, direct_x0=direct)
    seq_losses = []
    for sl, rs in wins:
        _, lo = seq.run_window(sl, rs)
        seq_losses.append(lo.cpu().numpy().copy())
    pip = trainer.Pipeline(g, feats, labels, cfg, direct_x0=direct)
    pip_losses = [lo.cpu().numpy().copy() for _, lo in pip.run_windows(wins)]
    assert np.array_equal(seq.model.flat.cpu().numpy(), pip.model.flat.cpu().numpy())
    for a, b in zip(seq_losses, pip_losses):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("arch", ["sage", "gin", "gcn"])
def test_batch_gradients_match_oracle(cfg1_graph, arch):
    """One 3-layer batch: every layer's dW / db against the oracle within 1e-5
    of the gradient's scale (fp32 sums of ~28K rows; multi-step weight
    trajectories of the all-rows GIN / SAGE layouts additionally see ReLU
    mask flips of near-zero activations, so they are checked per step)."""
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    dims, fan = (128, 32, 16, 4), [6, 4, 3]
    rng = np.random.default_rng(1)
    feats = rng.standard_normal((g.num_nodes, dims[0])).astype(np.float32)
    labels = rng.integers(0, dims[-1], size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=dims, fanouts=fan, arch=arch, batch_size=512, window_n=1, lr=0.1, seed=3)
    pipe = trainer.Pipeline(g, feats, labels, cfg, trainer.PipelineFlags(reorder=False))
    params = oracle.init_params(dims, 3)
    seeds = rng.choice(g.num_nodes, 512, replace=False)
    rs = oracle.derive_seed(3, 13, 0)
    _, losses = pipe.run_window([seeds], [rs])
    got = pipe.model.grads_numpy()
    b = oracle.sample_khop(g, seeds, fan, rs)
    _, seed_locals, _, csr = oracle.prepare_batch(b, arch)
    out, caches = oracle.forward(feats[b.unique_nodes.astype(np.int64)], csr, params, arch)
    loss, dl = oracle.softmax_xent(out[seed_locals], labels[b.seeds.astype(np.int64)])
    assert float(losses.cpu().numpy()[0]) / len(seeds) == pytest.approx(loss, rel=1e-5)
    dout = np.zeros_like(out)
    dout[seed_locals] = dl
    want = oracle.backward(dout, caches, csr, params, arch)
    for (gw, gb), (ww, wb) in zip(got, want):
        np.testing.assert_allclose(gw, ww, rtol=1e-5, atol=1e-5 * float(np.abs(ww).max()))
        np.testing.assert_allclose(gb, wb, rtol=1e-5, atol=1e-5 * float(np.abs(wb).max()))


@pytest.mark.parametrize("arch,direct", [("gcn", True), ("gcn", False), ("gin", False), ("sage", False)])
def test_graph_replay_bit_identical(cfg1_graph, arch, direct, monkeypatch):
    """The per-batch chain replayed as CUDA graphs (fgl_capture_*) gives
    exactly the parameters and losses of eager launches, and graphs are used."""
    import ctypes
    from paper_2409_14939_b200 import _lib, trainer
    g = cfg1_graph
    rng = np.random.default_rng(11)
    feats = rng.standard_normal((g.num_nodes, 20)).astype(np.float32)
    labels = rng.integers(0, 4, size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=(20, 16, 16, 4), fanouts=[6, 4, 3], batch_size=200, window_n=4, lr=0.2,
                              arch=arch)
    wins = [([rng.choice(g.num_nodes, 200, replace=False) for _ in range(4)], [100 * w + j for j in range(4)])
            for w in range(5)]
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("FGL_GRAPH", mode)
        stats0 = (ctypes.c_int64 * 3)()
        _lib.call("fgl_capture_stats", ctypes.cast(stats0, ctypes.c_void_p))
        pipe = trainer.Pipeline(g, feats, labels, cfg, direct_x0=direct)
        losses = [lo.cpu().numpy().copy() for _, lo in pipe.run_windows(wins)]
        stats1 = (ctypes.c_int64 * 3)()
        _lib.call("fgl_capture_stats", ctypes.cast(stats1, ctypes.c_void_p))
        out[mode] = (pipe.model.flat.cpu().numpy(), losses, stats1[0] - stats0[0], pipe.graph_fallbacks)
    assert out["0"][2] == 0
    assert out["1"][2] >= 5  # graph launches (window chains, prepare, sampler); a few may fall back
    assert np.array_equal(out["0"][0], out["1"][0])
    for a, b in zip(out["0"][1], out["1"][1]):
        assert np.array_equal(a, b)
