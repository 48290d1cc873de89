# A/B of GEMM kernel choices on the full serving step (bench.py, no SLO/cpu legs)
for cfg in "VOX_GEMM_MC=0" "VOX_GEMM_MC_BUDGET_KB=200" "VOX_GEMM_MC_BUDGET_KB=100" "VOX_GEMM_MC_BUDGET_KB=150"; do
  env $cfg timeout 300 python bench.py --no-slo --no-cpu --no-roofline --steps 64 --warmup 8 > gpurun_out/ab.json 2>/dev/null
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['ms_per_step'])")"
done
