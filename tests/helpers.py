"""Shared helpers for the test-suite (imported as ``helpers``)."""

import numpy as np


def golden_graph(store, name):
    import oracle
    off = store[f"g_{name}_off"].astype(np.int64)
    col = store[f"g_{name}_col"]
    n = len(off) - 1
    src = np.repeat(np.arange(n), np.diff(off))
    w = store[f"g_{name}_w"] if f"g_{name}_w" in store.files else None
    g = oracle.graph_from_edges(n, src, col, w)
    assert np.array_equal(g.row_offsets, store[f"g_{name}_off"])
    return g


def golden_layers(store, prefix, hops):
    return [(store[f"{prefix}_t{i}"], store[f"{prefix}_s{i}"], store[f"{prefix}_w{i}"]) for i in range(hops)]


def oracle_graph(dg):
    """The oracle's view of a device graph: int64 offsets, uint32 columns (IDs
    < 2^31; uint32 keeps numpy's promotions with the uint64 seeds exact and
    halves the host copy of a papers100M-shaped graph)."""
    import oracle
    off = dg.row_offsets.cpu().numpy()
    col = dg.col_indices.cpu().numpy().view(np.uint32)
    w = None if dg.edge_weights is None else dg.edge_weights.cpu().numpy()
    return oracle.CSRGraph(dg.num_nodes, off, col, None, None, w)


_POOL = {}


def _oracle_one(job):
    import oracle
    seeds, fan, rs = job
    return oracle.sample_khop(_POOL["g"], seeds, fan, rs)


def oracle_sample_many(g, seed_lists, fanouts, rseeds, procs=None):
    """oracle.sample_khop for several batches, one forked worker per batch
    (the workers only run numpy; the graph is shared copy-on-write)."""
    import multiprocessing as mp
    import os
    jobs = [(np.asarray(s), list(fanouts), int(r)) for s, r in zip(seed_lists, rseeds)]
    _POOL["g"] = g
    if len(jobs) == 1:
        return [_oracle_one(jobs[0])]
    n = max(1, min(len(jobs), procs or os.cpu_count() or 1))
    with mp.get_context("fork").Pool(n) as pool:
        return pool.map(_oracle_one, jobs, chunksize=1)


def assert_window_batch_equal(win, b, want):
    """Batch b of a DeviceWindow against an oracle Batch: every hop's
    (targets, sources, weights), the sorted unique nodes, the Philox draws and
    (when the window keeps them) the local IDs = ranks in unique_nodes."""
    got = win.to_batch(b)
    assert len(got.layers) == len(want.layers)
    for h, ((t, s, w), (t2, s2, w2)) in enumerate(zip(got.layers, want.layers)):
        assert np.array_equal(t, t2.astype(np.uint64)), (b, h, "targets")
        assert np.array_equal(s, s2.astype(np.uint64)), (b, h, "sources")
        assert np.array_equal(w, w2), (b, h, "weights")
    assert np.array_equal(got.unique_nodes, want.unique_nodes.astype(np.uint64)), (b, "unique")
    assert win.draws(b) == want.draws, (b, "draws")
    if got.local_layers and not win.s.depth_layout:
        uniq = got.unique_nodes
        for (lt, ls, _), (t, s, _) in zip(got.local_layers, got.layers):
            assert np.array_equal(lt, np.searchsorted(uniq, t)), (b, "local targets")
            assert np.array_equal(ls, np.searchsorted(uniq, s)), (b, "local sources")
    return got


def rel_fro(a, b) -> float:
    """||a - b||_F / ||b||_F in float64 (0 when both are zero)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b))
    d = float(np.linalg.norm(a - b))
    return d / nb if nb > 0 else d


def assert_rel_fro(a, b, tol, what=""):
    """Tensor-level relative error (Frobenius norm) within `tol`: the
    north-star 1e-5 for fp32 gradients / parameters that are sums over ~10^5
    rows, where any two fp32 implementations (the reference's OpenBLAS sgemm
    included) differ element-wise in the last bits and in the ReLU mask of
    activations within rounding of zero."""
    r = rel_fro(a, b)
    assert r <= tol, f"{what}: relative Frobenius error {r:.3e} > {tol:g}"
    return r


def oracle_backward_masked(dout, caches, csr, params, arch, masks, fp64=False):
    """oracle.backward (trainer.py:212-228) with the ReLU masks of the hidden
    layers supplied by the caller (masks[i]: bool [n_local, d_out] of layer
    i, or None = the oracle's own z > 0).  Feeding the GPU forward's masks
    separates arithmetic parity from activations that sit within fp32
    rounding of zero: one such mask flip moves a 10^5-row weight gradient by
    ~1/sqrt(rows) in relative norm, for any pair of fp32 implementations.
    fp64=True evaluates the same backward in float64 (the exact answer the
    fp32 implementations approximate)."""
    import oracle
    grads = [None] * len(params)
    dt = np.float64 if fp64 else np.float32
    dx = np.asarray(dout, dtype=dt)
    last = len(params) - 1
    for i in range(last, -1, -1):
        _, h, z = caches[i]
        h = np.asarray(h, dtype=dt)
        if i == last:
            dz = dx
        else:
            m = (z > 0) if masks[i] is None else masks[i]
            dz = dx * m
        grads[i] = [h.T @ dz, dz.sum(axis=0)]
        dh = dz @ np.asarray(params[i][0], dtype=dt).T
        tip, tix, tw = csr[i][3:6]
        if fp64:
            import scipy.sparse as sp
            a_t = sp.csr_matrix((np.asarray(tw, np.float64), np.asarray(tix, np.int64), np.asarray(tip, np.int64)),
                                shape=(len(tip) - 1, dh.shape[0]))
            dx = a_t @ dh
        else:
            dx = oracle.aggregate(tip, tix, tw, dh)
        if arch in ("gin", "sage"):
            dx = dx + dh
    return grads
