"""Time the layer-0 weight gradient alone (fgl_dense_bwd with dH = NULL, ReLU
mask from Z) at the products layer-0 shape; device time with CUDA events,
inputs larger than L2 rotated between calls.  Usage: wgrad_bench.py [n] [din] [dout]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib

n, din, dout = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (156000, 100, 64)))
ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
sets = []
for _ in range(3):
    H = torch.randn((n, ld(din)), device="cuda")
    Z = torch.randn((n, ld(dout)), device="cuda")
    dX = torch.randn((n, ld(dout)), device="cuda")
    sets.append((H, Z, dX))
W = torch.randn((din, dout), device="cuda") * 0.1
dW = torch.empty(din * dout + dout, device="cuda")
wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")


def bwd(i):
    H, Z, dX = sets[i % 3]
    _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(), ld(dout),
              Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0,
              ws.data_ptr(), wsb, st)


for i in range(5):
    bwd(i)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(30):
    bwd(i)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 30 * 1e3
byts = 4 * n * (ld(din) + 2 * ld(dout))
print(f"wgrad+reduce: n={n} {din}->{dout}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s", flush=True)
