"""Transposed-aggregation shape (products layer-1 backward): 130K rows with
0-3 edges (a few long rows) gathering 64-wide rows of a 16K-row dH; fgl_spmm
vs the software-pipelined fgl_spmm_gather kernel.  ncu-free: CUDA events."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2409_14939_b200 import _lib


def main():
    n, nsrc, d = 130_000, 16_000, 64
    rng = np.random.default_rng(0)
    lens = rng.choice([0, 1, 1, 1, 2, 2, 3], size=n)
    lens[rng.choice(n, 200, replace=False)] = rng.integers(9, 60, 200)
    ip = np.zeros(n + 1, np.int64); ip[1:] = np.cumsum(lens)
    ne = int(ip[-1])
    col = rng.integers(0, nsrc, ne).astype(np.int32)
    w = rng.random(ne).astype(np.float32)
    ipd, cd, wd = (torch.from_numpy(a).cuda() for a in (ip, col, w))
    X = torch.randn((nsrc, d), device="cuda")
    Ya = torch.empty((n, d), device="cuda"); Yb = torch.empty((n, d), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fns = {
        "spmm": lambda: _lib.call("fgl_spmm", ipd.data_ptr(), cd.data_ptr(), wd.data_ptr(), n, 0, X.data_ptr(), d,
                                  None, d, Ya.data_ptr(), d, d, st),
        "pipe": lambda: _lib.call("fgl_spmm_gather", ipd.data_ptr(), cd.data_ptr(), wd.data_ptr(), n, 0,
                                  X.data_ptr(), d, nsrc, Yb.data_ptr(), d, d, 16, st),
    }
    for name, fn in fns.items():
        ts = []
        for _ in range(15):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        print(f"{name}: {np.median(ts[3:]):.1f} us", flush=True)
    print("bit-exact:", torch.equal(Ya, Yb))


main()
