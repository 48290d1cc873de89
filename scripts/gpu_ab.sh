for e in VOX_ATTN_L2PF=0 VOX_ATTN_L2PF=2 VOX_ATTN_L2PF=4 VOX_ATTN_L2PF=8; do
  echo "== $e"
  env $e timeout 300 python scripts/trace_step.py --batch 224 --ctx 394 --steps 6 2>&1 | grep "span \|attn\[" | head -2
  env $e timeout 600 python bench.py --no-slo --no-cpu --no-roofline --no-cosy --no-csm > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'],d['detail']['lm_graph_step_ms'])"
done
