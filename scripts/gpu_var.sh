for tr in 1 ""; do
  VOX_BENCH_TRACE=$tr timeout 300 python bench.py --no-slo --no-cpu --no-roofline --steps 64 --warmup 8 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['ms_per_step'],d['detail'])"
  grep "trace: LM idle\|host iteration" gpurun_out/ab.err
done
