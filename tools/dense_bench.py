"""Time the dense kernels at the products layer-0 shape (device time, events).
Usage: python tools/dense_bench.py [n] [din] [dout]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib

n, din, dout = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (129000, 100, 64)))
ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
H = torch.randn((n, ld(din)), device="cuda")
W = torch.randn((din, dout), device="cuda") * 0.1
b = torch.randn(dout, device="cuda")
Z = torch.empty((n, ld(dout)), device="cuda")
dX = torch.randn((n, ld(dout)), device="cuda")
dH = torch.empty((n, ld(din)), device="cuda")
dW = torch.empty(din * dout + dout, device="cuda")
wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")


def fwd():
    _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout, Z.data_ptr(),
              ld(dout), 1, st)


def bwd():
    _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(), ld(dout),
              Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, dH.data_ptr(), ld(din),
              ws.data_ptr(), wsb, st)


for name, f in (("fwd", fwd), ("bwd(dW+db+dH)", bwd)):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = 4 * n * (din + dout) if name == "fwd" else 4 * n * (din + 2 * dout + din)
    print(f"{name}: n={n} {din}->{dout}: {ms*1e3:.1f} us, {byts/ms/1e6:.0f} GB/s", flush=True)
