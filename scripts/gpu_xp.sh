python -c "from paper_2602_00269_b200.build import build; build()"
VOX_GEMM_XPACKED_TEST=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_gemm.log
for xp in 0 1; do
 for bn in 128 256; do
 VOX_GEMM_XPACKED_TEST=$xp VOX_GEMM_BN_TEST=$bn timeout 300 python -c "
import sys, os; sys.path.insert(0,'.'); sys.path.insert(0,'baseline/_ref')
import numpy as np
os.environ['VOX_GEMM_PACKED_TEST']='1'
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice
dev=VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng=np.random.default_rng(0)
for name,(M,K) in {'qkv':(5120,3072),'o':(3072,3072),'gu':(16384,3072),'down':(3072,8192)}.items():
  w=rng.integers(0,65535,size=(M,K),dtype=np.uint16)&0x3FFF
  x=rng.integers(0,65535,size=(224,K),dtype=np.uint16)&0x3FFF
  res=[]
  for s in (1,2,3,4,6):
    _,ms=dev.gemm_test(w,x,None,s,iters=6)
    res.append((ms*1000,s))
  res.sort()
  print('xpacked $xp bn $bn', name, ' '.join('s%d %.1fus'%(s,t) for t,s in res[:3]))
" >> gpurun_out/xp.txt 2>&1
 done
done
