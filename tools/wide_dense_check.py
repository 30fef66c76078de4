import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2409_14939_b200 import _lib
ld=lambda d:(d+3)//4*4
st=torch.cuda.current_stream().cuda_stream
for n,din,dout in ((150000,602,64),(5000,602,64),(129,602,64),(3000,300,47),(2000,1000,128),(1500,64,172)):
    g=torch.Generator(device="cuda").manual_seed(n+din)
    H=torch.randn((n,ld(din)),device="cuda",generator=g); W=torch.randn((din,dout),device="cuda",generator=g)*0.05; b=torch.randn(dout,device="cuda",generator=g)
    Z=torch.full((n,ld(dout)),7.0,device="cuda")
    f=lambda: _lib.call("fgl_dense_fwd",H.data_ptr(),ld(din),n,din,W.data_ptr(),b.data_ptr(),dout,Z.data_ptr(),ld(dout),1,st)
    f(); torch.cuda.synchronize()
    ref=(H[:,:din].double()@W.double()+b.double()).clamp_min(0)
    err=((Z[:,:dout].double()-ref).abs().max()/ref.abs().max()).item()
    dZ=torch.randn((n,ld(dout)),device="cuda",generator=g); dH=torch.empty((n,ld(din)),device="cuda")
    _lib.call("fgl_dense_dgrad",dZ.data_ptr(),ld(dout),Z.data_ptr(),ld(dout),n,W.data_ptr(),din,dout,dH.data_ptr(),ld(din),st)
    torch.cuda.synchronize()
    refd=(dZ[:,:dout].double()*(Z[:,:dout]>0).double())@W.double().t()
    errd=((dH[:,:din].double()-refd).abs().max()/refd.abs().max()).item()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(n,din,dout,"fwd err %.2e dgrad err %.2e  fwd %.1f us" % (err, errd, e0.elapsed_time(e1)/10*1e3))
print("fallbacks", _lib.lib().fgl_dense_fallback_count())
