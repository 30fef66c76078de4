"""Input formats: the reference's MGL1 binary graph format
(graph.py:293-351) and from_edges (graph.py:151-183), against fixtures written
by the unmodified reference (tests/golden/make_golden.py graph_io).  The MGL1
read/write is host file IO (CPU test); the CSR build is the GPU path (-m gpu)."""

import io
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def _c1(golden):
    st = golden("graph_io")
    return st


def test_mgl1_load_matches_reference_file(golden):
    from paper_2409_14939_b200 import graph
    st = golden("graph_io")
    g = graph.load_binary(GOLD / "small_weighted.mgl1")
    assert g.num_nodes == 300 and g.num_edges == len(st["c1_src"])
    assert np.array_equal(g.row_offsets, st["c1_ro"]) and np.array_equal(g.col_indices, st["c1_ci"])
    assert np.array_equal(g.t_row_offsets, st["c1_tro"]) and np.array_equal(g.t_col_indices, st["c1_tci"])
    assert np.array_equal(g.edge_weights, st["c1_ew"]) and np.array_equal(g.t_edge_weights, st["c1_tew"])
    assert g.row_offsets.dtype == np.uint64 and g.edge_weights.dtype == np.float32


def test_mgl1_round_trip_bytes(tmp_path):
    from paper_2409_14939_b200 import graph
    g = graph.load_binary(GOLD / "small_weighted.mgl1")
    out = tmp_path / "rt.mgl1"
    graph.save_binary(g, out)
    assert out.read_bytes() == (GOLD / "small_weighted.mgl1").read_bytes()


def test_mgl1_format_errors(tmp_path):
    from paper_2409_14939_b200 import graph
    raw = (GOLD / "small_weighted.mgl1").read_bytes()
    bad = tmp_path / "bad.mgl1"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(graph.FormatError, match="bad magic"):
        graph.load_binary(bad)
    bad.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(graph.FormatError, match="truncated"):
        graph.load_binary(bad)
    bad.write_bytes(raw[:20])
    with pytest.raises(graph.FormatError, match="missing flag"):
        graph.load_binary(bad)


@pytest.mark.gpu
def test_from_edges_gpu_matches_reference(golden):
    from paper_2409_14939_b200 import graph
    st = golden("graph_io")
    for c in range(int(st["ncases"])):
        w = st[f"c{c}_w"] if f"c{c}_w" in st else None
        g = graph.from_edges(int(st[f"c{c}_n"]), st[f"c{c}_src"], st[f"c{c}_dst"], w)
        assert np.array_equal(g.row_offsets, st[f"c{c}_ro"]) and np.array_equal(g.col_indices, st[f"c{c}_ci"])
        assert np.array_equal(g.t_row_offsets, st[f"c{c}_tro"]) and np.array_equal(g.t_col_indices, st[f"c{c}_tci"])
        if w is not None:
            assert np.array_equal(g.edge_weights, st[f"c{c}_ew"]) and np.array_equal(g.t_edge_weights, st[f"c{c}_tew"])


@pytest.mark.gpu
def test_mgl1_without_transpose_rebuilds_on_gpu(golden, tmp_path):
    """A file whose transpose flag is 0 gets its transpose from the GPU build."""
    from paper_2409_14939_b200 import graph
    st = golden("graph_io")
    raw = (GOLD / "small_weighted.mgl1").read_bytes()
    n, m = 300, len(st["c1_src"])
    fwd = 4 + 16 + 2 + 8 * (n + 1) + 8 * m + 4 * m
    f = tmp_path / "fwd_only.mgl1"
    f.write_bytes(raw[:21] + b"\x00" + raw[22:fwd])
    g = graph.load_binary(f)
    assert np.array_equal(g.t_row_offsets, st["c1_tro"]) and np.array_equal(g.t_col_indices, st["c1_tci"])
    assert np.array_equal(g.t_edge_weights, st["c1_tew"]) and np.array_equal(g.col_indices, st["c1_ci"])


@pytest.mark.gpu
def test_from_edges_validation():
    from paper_2409_14939_b200 import graph
    from paper_2409_14939_b200.errors import ValidationError
    with pytest.raises(ValidationError, match="length mismatch"):
        graph.from_edges(4, [0, 1], [1])
    with pytest.raises(ValidationError, match="out of range"):
        graph.from_edges(4, [0, 5], [1, 2])
