"""Host-link roofline: pinned H2D copy bandwidth vs the zero-copy row gather
(fgl_gather_rows from pinned host memory) on products-like rows."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2409_14939_b200 import _lib

N, d = 2_450_000, 100
host = torch.empty((N, d), dtype=torch.float32).pin_memory()
host.uniform_()
dev = torch.empty((N, d), dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    e0.record(); dev.copy_(host, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"pinned H2D cudaMemcpy: {host.numel()*4/e0.elapsed_time(e1)/1e6:.1f} GB/s")
st = torch.cuda.current_stream().cuda_stream
for U in (100_000, 600_000):
    ids = torch.from_numpy(np.sort(np.random.default_rng(0).choice(N, U, replace=False)).astype(np.int32)).cuda()
    out = torch.empty((U, d), dtype=torch.float32, device="cuda")
    for _ in range(3):
        e0.record()
        _lib.call("fgl_gather_rows", host.data_ptr(), d, d, ids.data_ptr(), U, None, None, 0, None, d, out.data_ptr(), d, None, st)
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"zero-copy gather {U} rows x {d*4} B: {ms:.3f} ms = {U*d*4/ms/1e6:.1f} GB/s over the host link")
