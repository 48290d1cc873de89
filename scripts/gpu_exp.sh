set -x
python -c "from paper_2602_00269_b200.build import build; build()"
for kr in 0 1; do
 for bn in 128 256; do
  echo "KROT=$kr BN=$bn" >> gpurun_out/exp.txt
  VOX_GEMM_KROT=$kr VOX_GEMM_BN_TEST=$bn timeout 300 python -c "
import sys, os; sys.path.insert(0,'.'); sys.path.insert(0,'baseline/_ref')
import numpy as np
os.environ['VOX_GEMM_PACKED_TEST']='1'
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice
dev=VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng=np.random.default_rng(0)
for name,(M,K) in {'qkv':(5120,3072),'gu':(16384,3072),'down':(3072,8192)}.items():
  w=rng.integers(0,65535,size=(M,K),dtype=np.uint16)&0x3FFF
  x=rng.integers(0,65535,size=(224,K),dtype=np.uint16)&0x3FFF
  for s in (1,2,3):
    _,ms=dev.gemm_test(w,x,None,s,iters=8)
    print(name,'s',s,'%.1f us'%(ms*1000))
" >> gpurun_out/exp.txt 2>&1
 done
done
