python -c "from paper_2602_00269_b200.build import build; build()"
for pr in 1 0; do
 for bn in 128 256; do
  VOX_GEMM_PROBE=$pr VOX_GEMM_BN_TEST=$bn timeout 300 python -c "
import sys, os; sys.path.insert(0,'.'); sys.path.insert(0,'baseline/_ref')
import numpy as np
os.environ['VOX_GEMM_PACKED_TEST']='1'
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice
dev=VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng=np.random.default_rng(0)
M=2048
for K in (1024, 4096, 16384):
  w=rng.integers(0,65535,size=(M,K),dtype=np.uint16)&0x3FFF
  x=rng.integers(0,65535,size=(256,K),dtype=np.uint16)&0x3FFF
  _,ms=dev.gemm_test(w,x,None,1,iters=6)
  print('probe $pr bn $bn M',M,'N 256 K',K,'%.1f us'%(ms*1000), 'per-kb %.3f us'%(ms*1000/(K/64)), '%.0f TF'%(2*M*256*K/ms/1e9))
" >> gpurun_out/probe2.txt 2>&1
 done
done
