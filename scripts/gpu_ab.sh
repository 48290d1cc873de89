timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "VOX_GEMM_MC_BUDGET_KB=150" "VOX_GEMM_MC_BUDGET_KB=200"; do
  env $cfg timeout 300 python bench.py --no-slo --no-cpu --no-roofline --steps 64 --warmup 8 > gpurun_out/ab.json 2>/dev/null
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['ms_per_step'])")"
done
timeout 400 python scripts/trace_step.py --steps 4 2>&1 | grep -B3 -A12 "exposed"
