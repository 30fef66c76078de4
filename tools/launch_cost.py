"""Host cost of one C-ABI call that launches one tiny kernel (fgl_sgd on 64
floats), GPU otherwise idle: ctypes + cudaLaunchKernel floor."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib
p = torch.zeros(64, device="cuda"); g = torch.zeros(64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = _lib.lib().fgl_sgd
for _ in range(100):
    f(p.data_ptr(), g.data_ptr(), 64, 0.1, st)
torch.cuda.synchronize()
for n in (100, 1000):
    t = time.perf_counter()
    for _ in range(n):
        f(p.data_ptr(), g.data_ptr(), 64, 0.1, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{n} calls: {(t1 - t) / n * 1e6:.2f} us/call issue (raw ctypes fn)")
t = time.perf_counter()
for _ in range(1000):
    _lib.call("fgl_sgd", p.data_ptr(), g.data_ptr(), 64, 0.1, st)
print(f"_lib.call: {(time.perf_counter() - t) / 1000 * 1e6:.2f} us/call")
torch.cuda.synchronize()
