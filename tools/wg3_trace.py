"""Timeline of tc_wgrad3 (FGL_G3DBG=8, FGL_WGRAD=3): per-CTA globaltimer stamps."""
import os, sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["FGL_G3DBG"] = os.environ.get("FGL_G3DBG", "8")
os.environ["FGL_WGRAD"] = "3"
import numpy as np, torch
from paper_2409_14939_b200 import _lib
n, din, dout = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (156000, 100, 64)))
ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
H = torch.randn((n, ld(din)), device="cuda"); Z = torch.randn((n, ld(dout)), device="cuda")
dX = torch.randn((n, ld(dout)), device="cuda"); W = torch.randn((din, dout), device="cuda")
dW = torch.empty(din * dout + dout, device="cuda")
wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout); ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
for _ in range(3):
    _lib.call("fgl_dense_bwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dX.data_ptr(), ld(dout),
              Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0, ws.data_ptr(), wsb, st)
torch.cuda.synchronize()
buf = np.zeros(148 * 72, dtype=np.int64)
_lib.lib().fgl_debug_g3_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tr = buf.reshape(148, 72)
t0 = tr[:, 0].min()
f = lambda x: f"{(x - t0) / 1e3:6.2f}" if x else "   -  "
for c in (0, 1, 74, 147):
    r = tr[c]
    print(f"CTA {c}: start {f(r[0])} epi_start {f(r[70])} end {f(r[71])}")
    print("   producer issue:", " ".join(f(x) for x in r[58:66]))
    print("   mma cfull     :", " ".join(f(x) for x in r[50:58]))
    for j in range(8):
        v = r[2 + 6 * j: 8 + 6 * j]
        print(f"   tile {j} conv g0: full {f(v[0])} A+B {f(v[1])} cempty {f(v[2])} tst {f(v[3])} arrive {f(v[4])} empty {f(v[5])}")
print("kernel span", (tr[:, 71].max() - t0) / 1e3, "us")
