"""Dense layer kernels (tcgen05 3xTF32 path and SIMT fallback) against an fp64
numpy reference: forward act(HW+b), dgrad (dZ*mask)W^T, wgrad H^T dZ and db.
Tolerance: 1e-5 relative to the output scale (north star bar for fp32)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(1000, 100, 64), (4097, 64, 64), (300, 64, 47), (129, 47, 64), (777, 128, 172),
          (50, 12, 2), (5000, 602, 64), (3, 8, 16), (3000, 301, 47), (1500, 129, 64),
          (1024, 64, 172), (2000, 300, 200), (700, 64, 300), (2000, 1000, 128), (129, 1024, 16)]


def _ld(d):
    return (d + 3) // 4 * 4


def _pad(a):
    n, d = a.shape
    t = torch.zeros((n, _ld(d)), dtype=torch.float32, device="cuda")
    t[:, :d] = torch.from_numpy(a).cuda()
    return t


def _close(got, ref):
    scale = max(1e-6, float(np.abs(ref).max()))
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5 * scale)


@pytest.mark.parametrize("n,din,dout", SHAPES)
def test_forward_and_backward(n, din, dout):
    """Every shape runs on the tensor cores (wide inputs in K slices, wide
    outputs -- papers' 172 classes -- in N slices, the dgrad reduction in K
    slices): the SIMT fallback counter must not move."""
    from paper_2409_14939_b200 import _lib
    fb0 = _lib.lib().fgl_dense_fallback_count()
    rng = np.random.default_rng(n + din + dout)
    H = rng.standard_normal((n, din)).astype(np.float32)
    W = (rng.standard_normal((din, dout)) * 0.3).astype(np.float32)
    b = rng.standard_normal(dout).astype(np.float32)
    st = torch.cuda.current_stream().cuda_stream
    Hd, Wd, bd = _pad(H), torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    Z = torch.empty((n, _ld(dout)), dtype=torch.float32, device="cuda")
    for relu in (0, 1):
        _lib.call("fgl_dense_fwd", Hd.data_ptr(), _ld(din), n, din, Wd.data_ptr(), bd.data_ptr(), dout,
                  Z.data_ptr(), _ld(dout), relu, st)
        ref = H.astype(np.float64) @ W.astype(np.float64) + b
        if relu:
            ref = np.maximum(ref, 0)
        _close(Z[:, :dout].cpu().numpy(), ref)
    # backward with the ReLU mask of the layer output Z (relu=1 above)
    dX = rng.standard_normal((n, dout)).astype(np.float32)
    dXd = _pad(dX)
    mask = Z[:, :dout].cpu().numpy() > 0
    dW = torch.empty(din * dout + dout, dtype=torch.float32, device="cuda")
    dH = torch.empty((n, _ld(din)), dtype=torch.float32, device="cuda")
    wsb = _lib.lib().fgl_dense_bwd_ws_bytes(din, dout)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("fgl_dense_bwd", Hd.data_ptr(), _ld(din), n, din, Wd.data_ptr(), dout, dXd.data_ptr(),
              _ld(dout), Z.data_ptr(), _ld(dout), dW.data_ptr(), dW.data_ptr() + 4 * din * dout,
              dH.data_ptr(), _ld(din), ws.data_ptr(), wsb, st)
    dz = np.where(mask, dX, 0).astype(np.float64)
    _close(dW[: din * dout].cpu().numpy().reshape(din, dout), H.astype(np.float64).T @ dz)
    _close(dW[din * dout :].cpu().numpy(), dz.sum(0))
    _close(dH[:, :din].cpu().numpy(), dz @ W.astype(np.float64).T)
    # the chain's separate dgrad entry point (fgl_dense_dgrad)
    dH2 = torch.empty((n, _ld(din)), dtype=torch.float32, device="cuda")
    _lib.call("fgl_dense_dgrad", dXd.data_ptr(), _ld(dout), Z.data_ptr(), _ld(dout), n, Wd.data_ptr(), din, dout,
              dH2.data_ptr(), _ld(din), st)
    _close(dH2[:, :din].cpu().numpy(), dz @ W.astype(np.float64).T)
    if os.environ.get("FGL_DENSE", "") == "":
        assert _lib.lib().fgl_dense_fallback_count() == fb0, "a dense kernel took the SIMT fallback"


def test_simt_fallback_matches():
    """FGL_DENSE=simt forces the SIMT kernels; both paths meet the same bar."""
    code = "import sys; sys.argv=['x']; import pytest; sys.exit(pytest.main(['-q','-x','-m','gpu','tests/test_gpu_dense.py::test_forward_and_backward']))"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, FGL_DENSE="simt"), cwd=root,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]


def test_tc_dense4_bitidentical_to_tc_gemm3(tmp_path):
    """tc_dense4 (TMA boxes in the operand layout, the default for K, N <= 128)
    keeps tc_gemm3's rounding and MMA order: forward and dgrad outputs are
    bit-identical to the tc_gemm3 kernel (FGL_TC4=0) at the trainer's layer
    shapes, ragged row counts and a 47-wide output included."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tag, env in (("tc4", {}), ("tc3", {"FGL_TC4": "0"})):
        path = tmp_path / f"{tag}.npz"
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "tc4_check.py"), str(path)],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert "fallbacks 0" in r.stdout, r.stdout
        outs[tag] = np.load(path)
    for key in ("fwd_134000_100_64", "dgrad_134000_100_64", "fwd_16000_64_64", "dgrad_16000_64_64",
                "fwd_1000_64_47", "dgrad_1000_64_47", "fwd_77_100_64", "dgrad_77_100_64",
                "fwd_5000_128_128", "dgrad_5000_128_128", "fwd_3000_36_20"):
        a, b = outs["tc4"][key], outs["tc3"][key]
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), key
