"""Diagnostic: per-layer dW of one SAGE batch, GPU vs fp32 oracle vs fp64."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_2409_14939_b200 import trainer

arch = sys.argv[1] if len(sys.argv) > 1 else "sage"
dims = (128, 32, 16, 4)
fan = [6, 4, 3]
g = oracle.gen_power_law(100_000, 10, 1)
rng = np.random.default_rng(1)
feats = rng.standard_normal((g.num_nodes, dims[0])).astype(np.float32)
labels = rng.integers(0, dims[-1], size=g.num_nodes)
cfg = trainer.ModelConfig(layer_dims=dims, fanouts=fan, arch=arch, batch_size=512, window_n=1, lr=0.1, seed=3)
pipe = trainer.Pipeline(g, feats, labels, cfg, trainer.PipelineFlags(reorder=False))
params = oracle.init_params(dims, 3)
seeds = rng.choice(g.num_nodes, 512, replace=False)
rs = oracle.derive_seed(3, 13, 0)
pipe.run_window([seeds], [rs])
got = pipe.model.grads_numpy()
b = oracle.sample_khop(g, seeds, fan, rs)
tr, seed_locals, n, csr = oracle.prepare_batch(b, arch)
x0 = feats[b.unique_nodes.astype(np.int64)]
out, caches = oracle.forward(x0, csr, params, arch)
loss, dl = oracle.softmax_xent(out[seed_locals], labels[b.seeds.astype(np.int64)])
dout = np.zeros_like(out); dout[seed_locals] = dl
g32 = oracle.backward(dout, caches, csr, params, arch)
# fp64 dW from the same fp32 forward caches and dz chain
dx = dout.astype(np.float64)
for i in range(len(params) - 1, -1, -1):
    _, h, z = caches[i]
    dz = dx if i == len(params) - 1 else dx * (z > 0)
    dW64 = h.astype(np.float64).T @ dz
    dh = dz @ params[i][0].astype(np.float64).T
    dx = oracle.aggregate(*csr[i][3:6], dh.astype(np.float32)).astype(np.float64)
    if arch in ("gin", "sage"):
        dx = dx + dh
    e_gpu = np.abs(got[i][0] - dW64).max(); e_32 = np.abs(g32[i][0] - dW64).max()
    print(f"layer {i}: max|dW|={np.abs(dW64).max():.3e}  |gpu-fp64|={e_gpu:.3e}  |oracle32-fp64|={e_32:.3e}  |gpu-oracle32|={np.abs(got[i][0]-g32[i][0]).max():.3e}  rows={h.shape[0]}")
