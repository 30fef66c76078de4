"""Timeline of tc_gemm3 (FGL_G3DBG=8): per-CTA globaltimer stamps of each role."""
import os, sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["FGL_G3DBG"] = os.environ.get("FGL_G3DBG", "8")
import numpy as np, torch
from paper_2409_14939_b200 import _lib
n, din, dout = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (129000, 100, 64)))
ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
H = torch.randn((n, ld(din)), device="cuda"); W = torch.randn((din, dout), device="cuda"); b = torch.randn(dout, device="cuda")
Z = torch.empty((n, ld(dout)), device="cuda")
for _ in range(3):
    _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout, Z.data_ptr(), ld(dout), 1, st)
torch.cuda.synchronize()
buf = np.zeros(148 * 72, dtype=np.int64)
_lib.lib().fgl_debug_g3_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tr = buf.reshape(148, 72)
t0 = tr[:, 0][tr[:, 0] > 0].min()
for c in (0, 1, 74, 147):
    if tr[c, 0] == 0: continue
    r = tr[c]
    print(f"CTA {c}: start {(r[0]-t0)/1e3:.2f} prologue_done {(r[1]-t0)/1e3:.2f} end {(r[71]-t0)/1e3:.2f} us")
    for j in range(7):
        v = r[2 + 9 * j: 11 + 9 * j]
        if v[0] == 0: break
        print("   tile", j, " ".join(f"{nm}={(x-t0)/1e3:6.2f}" for nm, x in zip(("load", "conv0", "conv1", "mma", "epi0", "epi1", "staged", "bar", "copied"), v)))
print("tile-1 chunk CFULL seen by MMA (CTA 147):", " ".join(f"{(x - t0) / 1e3:6.2f}" for x in tr[147, 65:69]))
print("kernel span", (tr[:, 71].max() - t0) / 1e3, "us")
