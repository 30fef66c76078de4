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
