"""Dense forward / dgrad outputs at the trainer's layer shapes, saved for a
bitwise A/B between kernels (FGL_TC4=0 selects tc_gemm3) and checked against
fp64.  Usage: python tools/tc4_check.py out.npz"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2409_14939_b200 import _lib

ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
out = {}
worst = 0.0
for (n, din, dout, relu) in ((134000, 100, 64, 1), (16000, 64, 64, 1), (1000, 64, 47, 0), (77, 100, 64, 1),
                              (5000, 128, 128, 1), (3000, 36, 20, 0), (129, 602, 64, 1), (2000, 64, 172, 0)):
    g = torch.Generator(device="cuda").manual_seed(n + din)
    H = torch.randn((n, ld(din)), device="cuda", generator=g)
    W = torch.randn((din, dout), device="cuda", generator=g) * 0.1
    b = torch.randn(dout, device="cuda", generator=g)
    Z = torch.full((n, ld(dout)), 7.0, device="cuda")
    _lib.call("fgl_dense_fwd", H.data_ptr(), ld(din), n, din, W.data_ptr(), b.data_ptr(), dout, Z.data_ptr(),
              ld(dout), relu, st)
    ref = H[:, :din].double() @ W.double() + b.double()
    if relu:
        ref = ref.clamp_min(0)
    err = ((Z[:, :dout].double() - ref).abs().max() / ref.abs().max()).item()
    worst = max(worst, err)
    out[f"fwd_{n}_{din}_{dout}"] = Z.cpu().numpy()
    # dgrad: dH = (dZ * (Z > 0)) W^T
    dZ = torch.randn((n, ld(dout)), device="cuda", generator=g)
    dH = torch.full((n, ld(din)), 7.0, device="cuda")
    _lib.call("fgl_dense_dgrad", dZ.data_ptr(), ld(dout), Z.data_ptr(), ld(dout), n, W.data_ptr(), din, dout,
              dH.data_ptr(), ld(din), st)
    refd = (dZ[:, :dout].double() * (Z[:, :dout] > 0).double()) @ W.double().t()
    errd = ((dH[:, :din].double() - refd).abs().max() / refd.abs().max()).item()
    worst = max(worst, errd)
    out[f"dgrad_{n}_{din}_{dout}"] = dH.cpu().numpy()
    pad_ok = bool((Z[:, dout:] == 7.0).all() and (dH[:, din:] == 7.0).all())
    print(f"n {n:6d} din {din:3d} dout {dout:3d}: fwd rel err {err:.2e}  dgrad rel err {errd:.2e}  padding untouched {pad_ok}")
torch.cuda.synchronize()
print("fallbacks", _lib.lib().fgl_dense_fallback_count(), "worst", worst)
np.savez(sys.argv[1], **out)
