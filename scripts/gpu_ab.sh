for e in VOX_GEMM_L2PF=0 VOX_GEMM_L2PF=4 VOX_GEMM_L2PF=16; do
  echo "== $e"
  env $e timeout 300 python scripts/trace_step.py --batch 224 --ctx 394 --steps 6 2>&1 | grep "span " | head -1
  for i in 1 2; do env $e timeout 600 python bench.py --no-slo --no-cpu --no-roofline --no-cosy --no-csm > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'],d['detail']['lm_graph_step_ms'])"; done
done
