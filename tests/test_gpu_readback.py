"""Bit-exact read-back of the pipeline's intermediates (SURVEY 8(c) parity
items iii and iv; VERDICT r1 "next" #2): what ``Pipeline.prepare`` leaves in
HBM -- every model layer's block CSR, its stable transpose and the GCN /
GIN / GraphSAGE edge weights -- and the x0 feature blocks the Match loader
assembles, against ``oracle.prepare_batch`` (trainer.py:156-179) and
``feats[unique_nodes]`` (trainer.py:315).

Layouts: GCN runs the compact block layout (rows =
hop frontiers, columns = the next hop's frontier, model layer 0's columns =
window rows); GIN / GraphSAGE run depth-major window rows.  Each row of ours
is matched to the oracle's all-rows CSR row of the same global node."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

FAN = [8, 5, 3]
DIMS = (24, 16, 12, 5)


def _setup(cfg1_graph, arch, store="device", cache_ratio=0.0, match=True, nb=4, bs=400, seed=0):
    from paper_2409_14939_b200 import trainer
    g = cfg1_graph
    rng = np.random.default_rng(seed)
    feats = rng.standard_normal((g.num_nodes, DIMS[0])).astype(np.float32)
    labels = rng.integers(0, DIMS[-1], size=g.num_nodes)
    cfg = trainer.ModelConfig(layer_dims=DIMS, fanouts=FAN, arch=arch, batch_size=bs, window_n=nb, lr=0.1, seed=1)
    pipe = trainer.Pipeline(g, feats, labels, cfg, trainer.PipelineFlags(match=match), feature_store=store,
                            cache_ratio=cache_ratio)
    seeds = [rng.choice(g.num_nodes, bs, replace=False) for _ in range(nb)]
    rs = [oracle.derive_seed(1, 13, j) for j in range(nb)]
    win = pipe.sampler.sample(seeds, rs)
    win.host_counts()
    want = [oracle.sample_khop(g, s, FAN, r) for s, r in zip(seeds, rs)]
    return pipe, win, feats, want


def _rows_of(indptr, col, w, r0, r1):
    """Per-row (col, w) runs of rows [r0, r1) as python lists."""
    return [(col[indptr[r] : indptr[r + 1]], w[indptr[r] : indptr[r + 1]]) for r in range(r0, r1)]


def _oracle_rows(ip, ix, cw, uniq, ranks):
    """Oracle all-rows CSR rows of the given local ranks, sources as global IDs."""
    return [(uniq[ix[ip[k] : ip[k + 1]]].astype(np.int64), cw[ip[k] : ip[k + 1]]) for k in ranks]


@pytest.mark.parametrize("keep_l0_t", [False, True])
def test_prepare_block_csr_gcn(cfg1_graph, keep_l0_t):
    pipe, win, _, want = _setup(cfg1_graph, "gcn")
    pipe._keep_l0_transpose = keep_l0_t
    layers = pipe.prepare(win)
    import torch
    torch.cuda.synchronize()
    s = pipe.sampler
    H = len(FAN)
    front = s.frontier.cpu().numpy()
    uniq_all = s.unique.cpu().numpy()
    for b in range(win.num_batches):
        wb = want[b]
        uq = wb.unique_nodes.astype(np.int64)
        _, _, _, csr = oracle.prepare_batch(wb, "gcn")
        for h in range(H):
            i = H - 1 - h
            lay = layers[i]
            ip = lay["indptr"].cpu().numpy()
            e0, e1 = win.hop_edges(h)
            col = s.src_front[e0:e1].cpu().numpy()  # lay["col"] points here
            w = lay["w"][: e1 - e0].cpu().numpy()
            f0, f1 = win.front_range(h, b)
            tg = front[h * s.fcap + f0 : h * s.fcap + f1]
            ranks = np.searchsorted(uq, tg)
            nxt = (lambda c: front[(h + 1) * s.fcap + c]) if h + 1 < H else (lambda c: uniq_all[c])
            got = [(nxt(c), ww) for c, ww in _rows_of(ip, col, w, f0, f1)]
            o_ip, o_ix, o_cw, o_tip, o_tix, o_tw = csr[i]
            exp = _oracle_rows(o_ip, o_ix, o_cw, uq, ranks)
            for (gs, gw), (es, ew) in zip(got, exp):
                assert np.array_equal(gs, es) and np.array_equal(gw, ew), (b, h)
            # every oracle row outside the frontier is empty
            assert int(np.diff(o_ip)[ranks].sum()) == int(o_ip[-1])
            if lay["t_indptr"] is None:
                assert h == H - 1 and not keep_l0_t
                continue
            tip = lay["t_indptr"].cpu().numpy()
            tcol = lay["t_col"][: e1 - e0].cpu().numpy()
            tw = lay["t_w"][: e1 - e0].cpu().numpy()
            if h + 1 < H:
                q0, q1 = win.front_range(h + 1, b)
                src_nodes = front[(h + 1) * s.fcap + q0 : (h + 1) * s.fcap + q1]
            else:
                q0, q1 = win.unique_range(b)
                src_nodes = uniq_all[q0:q1]
            t_ranks = np.searchsorted(uq, src_nodes)
            got_t = [(front[h * s.fcap + c], ww) for c, ww in _rows_of(tip, tcol, tw, q0, q1)]
            exp_t = _oracle_rows(o_tip, o_tix, o_tw, uq, t_ranks)
            for (gs, gw), (es, ew) in zip(got_t, exp_t):
                assert np.array_equal(gs, es) and np.array_equal(gw, ew), (b, h, "transpose")
            assert int(np.diff(o_tip)[t_ranks].sum()) == int(o_tip[-1])


@pytest.mark.parametrize("arch", ["gin", "sage"])
def test_prepare_depth_layout_csr(cfg1_graph, arch):
    """GIN / GraphSAGE: forward rows (sources in CSR order and weights)
    identical to the oracle's all-rows CSR for every row of the layer's
    prefix; transposed rows hold the same (target, weight) multiset (their
    order follows the grouped forward CSR)."""
    import torch
    pipe, win, _, want = _setup(cfg1_graph, arch)
    layers = pipe.prepare(win)
    torch.cuda.synchronize()
    H = len(FAN)
    uniq_all = pipe.sampler.unique.cpu().numpy()
    for h in range(H):
        i = H - 1 - h
        lay = layers[i]
        ip = lay["indptr"].cpu().numpy()
        e0, e1 = win.hop_edges(h)
        col = pipe._bufs[f"colg{h}s0"][: e1 - e0].cpu().numpy()
        w = lay["w"][: e1 - e0].cpu().numpy()
        has_t = lay["t_indptr"] is not None
        if has_t:
            tip = lay["t_indptr"].cpu().numpy()
            tcol = lay["t_col"][: e1 - e0].cpu().numpy()
            tw = lay["t_w"][: e1 - e0].cpu().numpy()
        for b in range(win.num_batches):
            wb = want[b]
            uq = wb.unique_nodes.astype(np.int64)
            _, _, _, csr = oracle.prepare_batch(wb, arch)
            o_ip, o_ix, o_cw, o_tip, o_tix, o_tw = csr[i]
            u0, u1 = win.unique_range(b)
            p1 = u0 + win.prefix_rows(i, b)
            rows = uniq_all[u0:p1]
            exp = _oracle_rows(o_ip, o_ix, o_cw, uq, np.searchsorted(uq, rows))
            for (c, gw), (es, ew) in zip(_rows_of(ip, col, w, u0, p1), exp):
                assert np.array_equal(uniq_all[c], es) and np.array_equal(gw, ew), (b, h)
            assert int(np.diff(o_ip)[np.searchsorted(uq, rows)].sum()) == int(o_ip[-1])
            if not has_t:
                continue
            srcs = uniq_all[u0:u1]
            exp_t = _oracle_rows(o_tip, o_tix, o_tw, uq, np.searchsorted(uq, srcs))
            for (c, gw), (es, ew) in zip(_rows_of(tip, tcol, tw, u0, u1), exp_t):
                got_pairs = sorted(zip(uniq_all[c].tolist(), gw.tolist()))
                assert got_pairs == sorted(zip(es.tolist(), ew.tolist())), (b, h, "transpose")


@pytest.mark.parametrize("arch,store,cache,match", [
    ("gcn", "device", 0.0, True), ("gcn", "host", 0.0, True), ("gcn", "host", 0.15, True),
    ("gcn", "host", 0.0, False), ("gcn", "host", 0.15, False), ("gin", "host", 0.0, True),
    ("sage", "device", 0.0, True), ("sage", "host", 0.1, True)])
def test_x0_blocks_bit_exact(cfg1_graph, arch, store, cache, match):
    """Every batch's x0 block in schedule order -- Match rows copied from the
    previous batch's block (also through the depth-major row map), static
    HBM cache rows, HBM / pinned-host store rows -- equals
    feats[unique_nodes] bit for bit, and the per-position store / cache row
    counts equal the reference's simulate_epoch_io accounting."""
    import torch
    pipe, win, feats, want = _setup(cfg1_graph, arch, store, cache, match)
    nb = win.num_batches
    order = pipe.schedule(win, nb)
    pipe.loaded.zero_()
    pipe.cache_hits.zero_()
    uniq_all = pipe.sampler.unique
    for j, b in enumerate(order):
        prev = order[j - 1] if (j > 0 and match) else None
        x0 = pipe._gather_x0(win, b, prev, j, j % 2)
        u0, u1 = win.unique_range(b)
        rows = uniq_all[u0:u1].long().cpu().numpy()
        got = x0[: (u1 - u0) * pipe.ldf].view(u1 - u0, pipe.ldf)[:, : DIMS[0]].cpu().numpy()
        assert np.array_equal(got, feats[rows]), (j, b)
        assert np.array_equal(np.sort(rows), want[b].unique_nodes.astype(np.int64))
    torch.cuda.synchronize()
    o_order, ex, loads, _ = oracle.window_schedule([w.unique_nodes for w in want], True, DIMS[0])
    assert order == o_order
    deg = np.diff(cfg1_graph.row_offsets.astype(np.int64))
    mask = oracle.cache_mask(cfg1_graph.num_nodes, cache, deg)
    h2d, _, ch = oracle.epoch_h2d_bytes([ex], [loads], DIMS[0], match=match, cached=mask)
    assert int(pipe.loaded.sum().item()) * 4 * DIMS[0] == h2d
    assert int(pipe.cache_hits.sum().item()) * 4 * DIMS[0] == ch
