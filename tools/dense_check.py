"""Print max relative errors of the dense kernels vs fp64 numpy for a few shapes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2409_14939_b200 import _lib


def ld(d):
    return (d + 3) // 4 * 4


def pad(a):
    t = torch.zeros((a.shape[0], ld(a.shape[1])), dtype=torch.float32, device="cuda")
    t[:, : a.shape[1]] = torch.from_numpy(a).cuda()
    return t


def err(got, ref):
    s = max(1e-6, float(np.abs(ref).max()))
    return float(np.abs(got - ref).max() / s)


st = torch.cuda.current_stream().cuda_stream
for (n, din, dout) in [(1000, 100, 64), (300, 64, 47), (129, 47, 64), (5000, 64, 64), (777, 128, 172), (3, 8, 16)]:
    rng = np.random.default_rng(n)
    H = rng.standard_normal((n, din)).astype(np.float32)
    W = (rng.standard_normal((din, dout)) * 0.3).astype(np.float32)
    b = rng.standard_normal(dout).astype(np.float32)
    Hd, Wd, bd = pad(H), torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    Z = torch.empty((n, ld(dout)), dtype=torch.float32, device="cuda")
    _lib.call("fgl_dense_fwd", Hd.data_ptr(), ld(din), n, din, Wd.data_ptr(), bd.data_ptr(), dout, Z.data_ptr(), ld(dout), 1, st)
    ref = np.maximum(H.astype(np.float64) @ W + b, 0)
    zf = Z[:, :dout].cpu().numpy()
    e_fwd = err(zf, ref)
    bad = np.argwhere(np.abs(zf - ref) > 1e-4 * np.abs(ref).max())
    dX = rng.standard_normal((n, dout)).astype(np.float32)
    dXd = pad(dX)
    mask = zf > 0
    dW = torch.empty(din * dout + dout, dtype=torch.float32, device="cuda")
    dH = torch.empty((n, ld(din)), dtype=torch.float32, device="cuda")
    wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("fgl_dense_bwd", Hd.data_ptr(), ld(din), n, din, Wd.data_ptr(), dout, dXd.data_ptr(), ld(dout),
              Z.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, dH.data_ptr(), ld(din),
              ws.data_ptr(), wsb, st)
    dz = np.where(mask, dX, 0).astype(np.float64)
    e_dw = err(dW[: din * dout].cpu().numpy().reshape(din, dout), H.astype(np.float64).T @ dz)
    e_db = err(dW[din * dout:].cpu().numpy(), dz.sum(0))
    e_dh = err(dH[:, :din].cpu().numpy(), dz @ W.T)
    print(f"n={n} din={din} dout={dout}: fwd {e_fwd:.2e} (bad {len(bad)}, first {bad[:3].tolist()}) dW {e_dw:.2e} db {e_db:.2e} dH {e_dh:.2e}", flush=True)
