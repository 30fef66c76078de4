"""Short-row SpMM (fgl_spmm_gather, the layer-0 aggregation over the sampled
block graph: the lean high-occupancy kernel shared with fgl_spmm)
against the oracle's aggregation
(oracle/minigl_oracle.py aggregate, compute.py:164-185) and against fgl_spmm:
bit-exact, including empty rows, ragged tails, rows longer than the fast path
and column offsets (col_base)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ld(d):
    return (d + 3) // 4 * 4


def _csr(rng, n, max_len, n_src, long_rows=0):
    lens = rng.integers(0, max_len + 1, n)
    if long_rows:
        lens[rng.choice(n, long_rows, replace=False)] = max_len * 3 + 1
    indptr = np.zeros(n + 1, np.int64)
    indptr[1:] = np.cumsum(lens)
    col = rng.integers(0, n_src, int(indptr[-1])).astype(np.int32)
    w = rng.standard_normal(int(indptr[-1])).astype(np.float32)
    return indptr, col, w


def _run(name, indptr, col, w, X, d, col_base=0, max_len=5):
    from paper_2409_14939_b200 import _lib
    n = len(indptr) - 1
    ld = X.shape[1]
    ip, cd, wd = (torch.from_numpy(a).cuda() for a in (indptr, col + col_base, w))
    Y = torch.full((n, _ld(d)), float("nan"), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    if name == "gather":
        _lib.call("fgl_spmm_gather", ip.data_ptr(), cd.data_ptr(), wd.data_ptr(), n, col_base, X.data_ptr(), ld,
                  X.shape[0], Y.data_ptr(), _ld(d), d, max_len, st)
    else:
        _lib.call("fgl_spmm", ip.data_ptr(), cd.data_ptr(), wd.data_ptr(), n, col_base, X.data_ptr(), ld, None, ld,
                  Y.data_ptr(), _ld(d), d, st)
    torch.cuda.synchronize()
    return Y[:, :d].cpu().numpy()


@pytest.mark.parametrize("n,d,max_len,long_rows", [
    (1, 100, 5, 0), (17, 100, 5, 0), (5000, 100, 5, 0), (3001, 47, 10, 0), (2000, 64, 15, 0),
    (4000, 100, 5, 7), (333, 128, 1, 0), (1000, 256, 3, 2), (64, 8, 16, 0)])
def test_gather_matches_oracle_and_spmm(n, d, max_len, long_rows):
    from oracle.minigl_oracle import aggregate
    rng = np.random.default_rng(n * 7 + d + max_len)
    n_src = 20000
    indptr, col, w = _csr(rng, n, max_len, n_src, long_rows)
    feats = rng.standard_normal((n_src, d)).astype(np.float32)
    X = torch.zeros((n_src, _ld(d)), dtype=torch.float32, device="cuda")
    X[:, :d] = torch.from_numpy(feats).cuda()
    got = _run("gather", indptr, col, w, X, d, max_len=max_len)
    ref = _run("spmm", indptr, col, w, X, d)
    assert np.array_equal(got, ref)
    if n <= 5000:
        assert np.array_equal(got, aggregate(indptr, col, w, feats))


def test_gather_col_base_and_empty():
    rng = np.random.default_rng(3)
    indptr = np.zeros(40, np.int64)  # 39 empty rows
    X = torch.randn((100, 100), device="cuda")
    got = _run("gather", indptr, np.zeros(0, np.int32), np.zeros(0, np.float32), X, 100)
    assert np.array_equal(got, np.zeros((39, 100), np.float32))
    indptr, col, w = _csr(rng, 500, 5, 50)
    a = _run("gather", indptr, col, w, X, 100, col_base=37)
    b = _run("spmm", indptr, col, w, X, 100, col_base=37)
    assert np.array_equal(a, b)


def test_gather_rejects_long_rows_and_wide_rows():
    from paper_2409_14939_b200 import _lib
    from paper_2409_14939_b200.errors import ConfigError, ValidationError
    X = torch.zeros((10, 300), device="cuda")
    Y = torch.zeros((1, 300), device="cuda")
    ip = torch.zeros(2, dtype=torch.int64, device="cuda")
    with pytest.raises(ValidationError):
        _lib.call("fgl_spmm_gather", ip.data_ptr(), None, None, 1, 0, X.data_ptr(), 300, 10, Y.data_ptr(), 300,
                  300, 5, 0)
    with pytest.raises(ConfigError):
        _lib.call("fgl_spmm_gather", ip.data_ptr(), None, None, 1, 0, X.data_ptr(), 100, 10, Y.data_ptr(), 100,
                  100, 17, 0)
