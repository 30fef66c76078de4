"""Dense kernels' fixed cost vs per-row cost: device time of fgl_dense_fwd /
fgl_dense_dgrad / fgl_dense_bwd over row counts and CTA budgets (events,
back-to-back launches).  Usage: python tools/dense_sweep.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib

ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
L = _lib.lib()


def timeit(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for din, dout in ((100, 64), (64, 64)):
    for n in (1024, 16000, 64000, 134000):
        H = torch.randn((n, ld(din)), device="cuda")
        W = torch.randn((din, dout), device="cuda") * 0.1
        b = torch.randn(dout, device="cuda")
        Z = torch.randn((n, ld(dout)), device="cuda")
        dX = torch.randn((n, ld(dout)), device="cuda")
        dH = torch.empty((n, ld(din)), device="cuda")
        dW = torch.empty(din * dout + dout, device="cuda")
        wsb = L.fgl_dense_bwd_ws_bytes(din, dout)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        fwd = lambda: _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout,
                                Z.data_ptr(), ld(dout), 1, st)
        wg = lambda: _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(),
                               ld(dout), Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0,
                               ws.data_ptr(), wsb, st)
        dg = lambda: _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(),
                               ld(dout), Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout,
                               dH.data_ptr(), ld(din), ws.data_ptr(), wsb, st)
        for ctas in (148, 74):
            L.fgl_set_dense_ctas(ctas)
            bf = 4 * n * (din + dout)
            tf, tw, tb = timeit(fwd), timeit(wg), timeit(dg)
            print(f"din {din} dout {dout} n {n:6d} ctas {ctas:3d}: fwd {tf:6.1f} us ({bf / tf / 1e3:5.0f} GB/s)  "
                  f"wgrad {tw:6.1f} us  wgrad+dgrad {tb:6.1f} us", flush=True)
L.fgl_set_dense_ctas(0)
