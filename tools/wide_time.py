"""Device time of fgl_dense_fwd / fgl_dense_dgrad at given shapes (CUDA graph of
10 calls): python tools/wide_time.py n:din:dout[:d] ...  (":d" = dgrad, ":w" = wgrad)"""
import sys; sys.path.insert(0, '.')
import torch
from paper_2409_14939_b200 import _lib
ld = lambda d: (d + 3) // 4 * 4
cs = lambda: torch.cuda.current_stream().cuda_stream
for spec in sys.argv[1:]:
    parts = spec.split(":")
    n, din, dout = (int(x) for x in parts[:3])
    mode = parts[3] if len(parts) > 3 else ""
    dg = mode == "d"
    H = torch.randn((n, ld(din)), device="cuda"); W = torch.randn((din, dout), device="cuda") * 0.05
    b = torch.randn(dout, device="cuda"); Z = torch.randn((n, ld(dout)), device="cuda")
    dZ = torch.randn((n, ld(dout)), device="cuda")
    if mode == "w":  # weight gradient only (dW, db; no dH)
        dW = torch.empty(din * dout + dout, device="cuda")
        wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        f = lambda: _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dZ.data_ptr(),
                              ld(dout), Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, 0,
                              ld(din), ws.data_ptr(), wsb, cs())
        byts = 4 * n * (ld(din) + 2 * ld(dout))
    elif dg:
        f = lambda: _lib.call("fgl_dense_dgrad", dZ.data_ptr(), ld(dout), Z.data_ptr(), ld(dout), n, W.data_ptr(), din,
                              dout, H.data_ptr(), ld(din), cs())
        byts = 4 * n * (ld(din) + 2 * ld(dout))
    else:
        f = lambda: _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout,
                              Z.data_ptr(), ld(dout), 1, cs())
        byts = 4 * n * (ld(din) + ld(dout))
    for _ in range(3): f()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10): f()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    print(f"{spec}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s", flush=True)
