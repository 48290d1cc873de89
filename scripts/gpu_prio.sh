python -c "from paper_2602_00269_b200.build import build; build()"
for pr in 0 1 0 1; do
  VOX_STREAM_PRIO=$pr timeout 300 python bench.py --no-slo --no-cpu --no-roofline > gpurun_out/bench_prio$pr.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_prio$pr.json').read().strip().splitlines()[-1]); print('prio $pr', d['value'], d['ms_per_step'], d['detail']['lm_graph_step_ms'])" >> gpurun_out/prio.txt
done
timeout 240 python scripts/cublas_ref.py > gpurun_out/cublas.txt 2>&1
