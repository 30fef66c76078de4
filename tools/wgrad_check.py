"""Weight gradient [dW; db] of fgl_dense_bwd (tc_wgrad5 or, with FGL_WGRAD5=0,
tc_wgrad3) against fp64 at the trainer's layer shapes, plus device time of
the call (CUDA graph of 20 launches).  Usage: python tools/wgrad_check.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib

ld = lambda d: (d + 3) // 4 * 4
L = _lib.lib()
for n, din, dout in ((134000, 100, 64), (16000, 64, 64), (1000, 64, 47), (77, 100, 64), (3000, 36, 20), (50000, 127, 64)):
    g = torch.Generator(device="cuda").manual_seed(n + din)
    H = torch.randn((n, ld(din)), device="cuda", generator=g)
    Z = torch.randn((n, ld(dout)), device="cuda", generator=g)
    dX = torch.randn((n, ld(dout)), device="cuda", generator=g)
    W = torch.randn((din, dout), device="cuda", generator=g)
    dW = torch.zeros(din * dout + dout, device="cuda")
    wsb = L.fgl_dense_bwd_ws_bytes(din, dout)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")

    def f(st):
        _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(), ld(dout),
                  Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0, ws.data_ptr(), wsb,
                  st)
    f(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dz = dX[:, :dout].double() * (Z[:, :dout] > 0).double()
    refW = H[:, :din].double().t() @ dz
    refb = dz.sum(0)
    gw = dW[: din * dout].view(din, dout).double()
    gb = dW[din * dout:].double()
    ew = ((gw - refW).abs().max() / refW.abs().max()).item()
    eb = ((gb - refb).abs().max() / refb.abs().max()).item()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f(s.cuda_stream)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            f(s.cuda_stream)
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e3
    byts = 4 * n * (din + 2 * dout)
    print(f"n {n:6d} din {din:3d} dout {dout:3d}: dW rel err {ew:.2e}  db rel err {eb:.2e}  {t:6.1f} us "
          f"({byts / t / 1e3:5.0f} GB/s)", flush=True)
print("fallbacks", L.fgl_dense_fallback_count())
