"""Time fgl_spmm vs fgl_spmm_gather on a layer-0-shaped aggregation: random
rows of <= fan edges gathering d-wide rows from a products-sized feature
table (2.45M x 100 fp32, larger than L2).  CUDA events, median of reps."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_14939_b200 import _lib  # noqa: E402


def main():
    n_src, d = 2_449_029, 100
    X = torch.randn((n_src, d), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for n, fan in ((134_000, 5), (400_000, 5), (120_000, 8), (120_000, 10)):
        lens = torch.randint(fan // 2, fan + 1, (n,), device="cuda")
        ip = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        ip[1:] = torch.cumsum(lens, 0)
        ne = int(ip[-1])
        col = torch.randint(0, n_src, (ne,), device="cuda", dtype=torch.int32)
        w = torch.rand(ne, device="cuda")
        Ya = torch.empty((n, d), device="cuda")
        Yb = torch.empty((n, d), device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

        def spmm():
            _lib.call("fgl_spmm", ip.data_ptr(), col.data_ptr(), w.data_ptr(), n, 0, X.data_ptr(), d, None, d,
                      Ya.data_ptr(), d, d, st)

        def gather():
            _lib.call("fgl_spmm_gather", ip.data_ptr(), col.data_ptr(), w.data_ptr(), n, 0, X.data_ptr(), d, n_src,
                      Yb.data_ptr(), d, d, fan, st)

        coll = col.long()

        def raw():  # ceiling probe: torch's row gather of the same random rows (no arithmetic)
            torch.index_select(X, 0, coll)

        res = {}
        for name, fn in (("spmm", spmm), ("gather", gather), ("raw", raw)):
            ts = []
            for _ in range(15):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            res[name] = float(np.median(ts[3:]))
        same = torch.equal(Ya, Yb)
        gb = (ne * (d * 4 + 8) + n * (d * 4 + 8)) / 1e9
        raw_gb = ne * d * 4 * 2 / 1e9
        print(f"n={n} fan={fan} edges={ne}: spmm {res['spmm']:.1f} us ({gb / res['spmm'] * 1e6:.0f} GB/s)  "
              f"gather {res['gather']:.1f} us ({gb / res['gather'] * 1e6:.0f} GB/s)  bit-exact={same}  "
              f"raw index_select {res['raw']:.1f} us ({raw_gb / res['raw'] * 1e6:.0f} GB/s read+write)", flush=True)


if __name__ == "__main__":
    main()
