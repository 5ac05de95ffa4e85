import sys, ctypes, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_1109_5114_b200.bsf as bsf
bsf.LIB_PATH='tools/libbsf_dbg.so'
L=bsf.lib()
from test_gpu_parity import _small_smooth
from gpu_util import make_plan
w,img,cov=_small_smooth(45,53,3.0)
plan=make_plan(w,policy=1,order=2)
g=plan.empty_g(); plan.preintegrate(img.cuda(),g)
dump=torch.zeros(81*8,dtype=torch.float64,device='cuda')
L.bsf_debug_set_dump.argtypes=[ctypes.c_void_p]; L.bsf_debug_set_dump(dump.data_ptr())
pts=torch.tensor([[0,0,23]],dtype=torch.int32,device='cuda'); out=torch.empty(1,dtype=torch.float64,device='cuda')
plan.filter_points(g,cov.cuda(),pts,out); torch.cuda.synchronize()
np.save('gpurun_out/taps.npy',dump.cpu().numpy().reshape(81,8)); print(out.item())
