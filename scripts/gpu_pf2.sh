python -c "from paper_2602_00269_b200.build import build; build()"
for pf in 0 4 8 16; do
  echo "L2PF=$pf" >> gpurun_out/pf2.txt
  VOX_GEMM_L2PF=$pf SWEEP_MT=1 SWEEP_N=256 timeout 600 python scripts/gemm_sweep.py 2>&1 | grep -E "^(qkv|gu|down)" | cut -c1-120 >> gpurun_out/pf2.txt
  VOX_GEMM_L2PF=$pf timeout 300 python bench.py --no-slo --no-cpu --no-roofline > gpurun_out/bench_pf.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_pf.json').read().strip().splitlines()[-1]); print('bench l2pf $pf', d['value'], d['ms_per_step'], d['detail']['lm_graph_step_ms'])" >> gpurun_out/pf2.txt
done
