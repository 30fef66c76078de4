cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3c
for d in 0 32 2 1 4 33 6; do
  echo "== FGL_G3DBG=$d"; FGL_G3DBG=$d python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_2409_14939_b200 import _lib
L=_lib.lib(); st=torch.cuda.current_stream().cuda_stream
for n,din,dout in ((134000,100,64),(16000,64,64)):
  ld=lambda d:(d+3)//4*4
  H=torch.randn((n,ld(din)),device='cuda'); W=torch.randn((din,dout),device='cuda'); b=torch.randn(dout,device='cuda'); Z=torch.empty((n,ld(dout)),device='cuda')
  f=lambda: _lib.call("fgl_dense_fwd",H.data_ptr(),ld(din),n,din,W.data_ptr(),b.data_ptr(),dout,Z.data_ptr(),ld(dout),1,st)
  for c in (148,74):
    L.fgl_set_dense_ctas(c)
    for _ in range(3): f()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    print(n,din,dout,'ctas',c,'fwd us',round(e0.elapsed_time(e1)/20*1e3,1))
PY
done
