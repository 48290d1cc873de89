timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --batch 224 --ctx 394 --steps 6 2>&1 | grep "span \|gemm_mc\[128\]" | head -3
for i in 1 2 3; do timeout 600 python bench.py --no-slo --no-cpu --no-roofline --no-cosy --no-csm > gpurun_out/b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['ms_per_step'],d['detail']['lm_graph_step_ms'])"; done
