for e in X=1 VOX_GEMM_L2PF=48 VOX_GEMM_MC_MIN_ROWS=1 "VOX_GEMM_MC_MIN_ROWS=1 VOX_GEMM_L2PF=48"; do
  echo "== $e"
  env $e timeout 600 python bench.py --no-slo --no-cpu --no-cosy --no-csm > gpurun_out/b.json 2> gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value']);print([(p['batch'],p['ms_per_step']) for p in d['roofline']['batch_sweep']['points']])"
done
