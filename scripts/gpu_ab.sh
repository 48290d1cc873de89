timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "VOX_GEMM_RED=0" "VOX_GEMM_RED=1"; do
  env $cfg timeout 400 python scripts/trace_step.py --steps 4 2>&1 | grep -A10 "untraced\|exposed" | grep -v "boundaries\|->\|per kernel\|launches"
done
python bench.py --no-slo --no-cpu --no-roofline > gpurun_out/ab.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['ms_per_step'])"
