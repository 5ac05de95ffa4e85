import sys, os, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from test_gpu_parity import _small_smooth
from gpu_util import make_plan
from paper_1109_5114_b200 import bsf
w,img,cov=_small_smooth(45,53,3.0)
pts=torch.tensor([[0,0,23],[0,0,22],[0,1,23],[0,5,23]],dtype=torch.int32)
res={}
for prec in (bsf.BSF_PREC_DD, bsf.BSF_PREC_FP64):
    plan=make_plan(w,policy=1,order=2,precision=prec)
    f=img.cuda(); c=cov.cuda(); g=plan.empty_g(); plan.preintegrate(f,g)
    out=torch.empty(4,dtype=torch.float64,device='cuda'); aux=torch.empty(48,dtype=torch.float64,device='cuda')
    plan.filter_points_aux(g,c,pts.cuda(),out,aux); torch.cuda.synchronize()
    res['out%d'%prec]=out.cpu().numpy(); res['aux%d'%prec]=aux.cpu().numpy().reshape(4,12)
    res['g%d'%prec]=g.cpu().numpy()
np.savez('gpurun_out/dbg1.npz',**res)
print(res['out1'],res['out0']); print(res['aux1'])
