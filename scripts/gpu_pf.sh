python -c "from paper_2602_00269_b200.build import build; build()"
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_lm.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
for pf in 0 1 0 1; do
  VOX_GEMM_L2PF=$pf timeout 300 python bench.py --no-slo --no-cpu --no-roofline > gpurun_out/bench_pf$pf.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_pf$pf.json').read().strip().splitlines()[-1]); print('l2pf $pf', d['value'], d['ms_per_step'], d['detail']['lm_graph_step_ms'])" >> gpurun_out/pf.txt
done
