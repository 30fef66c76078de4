"""Static-degree HBM feature cache (memsim.py:110-186 made
real): host-link / cache / Match byte counts equal the reference's
simulate_epoch_io accounting (oracle.epoch_h2d_bytes with oracle.cache_mask,
itself pinned to the reference's golden io numbers), and the cache never
changes a feature row (x0 bit-exact -> identical training)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ratio,match", [(0.1, True), (0.25, True), (0.1, False), (0.0, True)])
def test_cache_window_io_matches_simulate_epoch_io(cfg1_graph, ratio, match):
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(21)
    d = 24
    feats = rng.standard_normal((g.num_nodes, d)).astype(np.float32)
    labels = rng.integers(0, 3, size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=(d, 16, 3), fanouts=[10, 5], batch_size=256, window_n=6,
                              lr=0.1, seed=0)
    flags = trainer.PipelineFlags(match=match)
    pipe = trainer.Pipeline(g, feats, labels, cfg, flags, feature_store="host", cache_ratio=ratio)
    seeds = [rng.choice(g.num_nodes, 256, replace=False) for _ in range(6)]
    rs = [oracle.derive_seed(0, 13, j) for j in range(6)]
    pipe.loaded.zero_()
    pipe.cache_hits.zero_()
    pipe.run_window(seeds, rs)
    batches = [oracle.sample_khop(g, s, [10, 5], r) for s, r in zip(seeds, rs)]
    _, ex, loads, _ = oracle.window_schedule([b.unique_nodes for b in batches], True, d)
    deg = np.diff(g.row_offsets.astype(np.int64))
    mask = oracle.cache_mask(g.num_nodes, ratio, deg)
    h2d, mt, ch = oracle.epoch_h2d_bytes([ex], [loads], d, match=match, cached=mask)
    assert int(pipe.loaded.sum().item()) * 4 * d == h2d
    assert int(pipe.cache_hits.sum().item()) * 4 * d == ch
    if ratio > 0:
        assert np.array_equal(pipe.cache.mask_numpy(g.num_nodes), mask)
    # the cache only changes where a row comes from, never its value
    ref = trainer.Pipeline(g, feats, labels, cfg, flags, feature_store="device")
    ref.run_window(seeds, rs)
    assert np.array_equal(ref.model.flat.cpu().numpy(), pipe.model.flat.cpu().numpy())


def test_train_reports_cache_bytes(golden_meta):
    """trainer.train(cache_ratio=...) reports the three byte counts per epoch."""
    from paper_2409_14939_b200 import trainer
    g, x, labels = oracle.two_cluster_task(200, 16, 0)
    cfg = trainer.ModelConfig(layer_dims=(16, 32, 2), fanouts=[4, 4], batch_size=40, window_n=3, epochs=2,
                              seed=0, lr=0.3)
    base = trainer.train(g, x, labels, cfg)
    rep = trainer.train(g, x, labels, cfg, cache_ratio=0.2)
    assert rep.losses == base.losses
    for e0, e1 in zip(base.epochs, rep.epochs):
        t0, t1 = e0.traffic, e1.traffic
        assert t1["bytes_served_by_cache"] > 0
        assert t1["bytes_host_to_device"] + t1["bytes_served_by_cache"] == t0["bytes_host_to_device"]
        assert t1["bytes_served_by_match"] == t0["bytes_served_by_match"]


def test_cache_validation():
    from paper_2409_14939_b200 import trainer
    from paper_2409_14939_b200.errors import ValidationError
    g, x, labels = oracle.two_cluster_task(50, 4, 0)
    cfg = trainer.ModelConfig(layer_dims=(4, 2), fanouts=[2], batch_size=10)
    with pytest.raises(ValidationError, match="cache_ratio"):
        trainer.Pipeline(g, x, labels, cfg, feature_store="host", cache_ratio=1.5)
    with pytest.raises(ValidationError, match="unknown cache policy"):
        trainer.Pipeline(g, x, labels, cfg, feature_store="host", cache_ratio=0.5, cache_policy="lru")
    with pytest.raises(ValidationError, match="host-resident"):
        trainer.Pipeline(g, x, labels, cfg, feature_store="device", cache_ratio=0.5)
