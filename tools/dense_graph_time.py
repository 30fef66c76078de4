"""Device time per dense launch without host overhead: 20 launches captured in
one CUDA graph, replayed.  Usage: python tools/dense_graph_time.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14939_b200 import _lib

ld = lambda d: (d + 3) // 4 * 4
L = _lib.lib()


def graph_time(f, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            f(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            f(s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


shapes = [(int(a), int(b), int(c)) for a, b, c in (x.split(",") for x in sys.argv[1:])] or \
    [(134000, 100, 64), (64000, 100, 64), (16000, 64, 64), (16000, 64, 47), (1024, 64, 47)]
for n, din, dout in shapes:
    H = torch.randn((n, ld(din)), device="cuda")
    W = torch.randn((din, dout), device="cuda") * 0.1
    b = torch.randn(dout, device="cuda")
    Z = torch.randn((n, ld(dout)), device="cuda")
    dX = torch.randn((n, ld(dout)), device="cuda")
    dH = torch.empty((n, ld(din)), device="cuda")
    dW = torch.empty(din * dout + dout, device="cuda")
    wsb = L.fgl_dense_bwd_ws_bytes(din, dout)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    fwd = lambda st: _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout,
                               Z.data_ptr(), ld(dout), 1, st)
    dg = lambda st: _lib.call("fgl_dense_dgrad", dX.data_ptr(), ld(dout), Z.data_ptr(), ld(dout), n, W.data_ptr(),
                              din, dout, dH.data_ptr(), ld(din), st)
    wg = lambda st: _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(),
                              ld(dout), Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0,
                              ws.data_ptr(), wsb, st)
    for ctas in (148, 74):
        L.fgl_set_dense_ctas(ctas)
        tf, td, tw = graph_time(fwd), graph_time(dg), graph_time(wg)
        bf = 4 * n * (din + dout)
        print(f"n {n:6d} din {din:3d} dout {dout:3d} ctas {ctas:3d}: fwd {tf:6.1f} us ({bf / tf / 1e3:5.0f} GB/s)  "
              f"dgrad {td:6.1f} us  wgrad(+reduce) {tw:6.1f} us", flush=True)
L.fgl_set_dense_ctas(0)
