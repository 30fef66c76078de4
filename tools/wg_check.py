import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2409_14939_b200 import _lib
ld = lambda d: (d + 3) // 4 * 4
st = torch.cuda.current_stream().cuda_stream
for n, din, dout in [(9600, 64, 48), (9611, 64, 48), (20000, 64, 47), (50000, 100, 64), (2000, 48, 32), (30000, 48, 32)]:
    rng = np.random.default_rng(n)
    H = rng.standard_normal((n, din)).astype(np.float32)
    dX = rng.standard_normal((n, dout)).astype(np.float32)
    Z = rng.standard_normal((n, dout)).astype(np.float32)
    def pad(a):
        t = torch.zeros((a.shape[0], ld(a.shape[1])), device="cuda"); t[:, :a.shape[1]] = torch.from_numpy(a).cuda(); return t
    Hd, dXd, Zd = pad(H), pad(dX), pad(Z)
    W = torch.zeros((din, dout), device="cuda")
    dW = torch.zeros(din * dout + dout, device="cuda")
    wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("fgl_dense_bwd", Hd.data_ptr(), ld(din), n, din, W.data_ptr(), dout, dXd.data_ptr(), ld(dout),
              Zd.data_ptr(), ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout, None, 0, ws.data_ptr(), wsb, st)
    torch.cuda.synchronize()
    dz = dX.astype(np.float64) * (Z > 0)
    ref = H.astype(np.float64).T @ dz
    rdb = dz.sum(0)
    got = dW[:din * dout].cpu().numpy().reshape(din, dout)
    gdb = dW[din * dout:].cpu().numpy()
    e1 = np.abs(got - ref).max() / np.abs(ref).max()
    e2 = np.abs(gdb - rdb).max() / np.abs(rdb).max()
    print(n, din, dout, f"dW rel err {e1:.2e}  db rel err {e2:.2e}", flush=True)
