set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 180 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_gemm.log
SWEEP_MT=1 SWEEP_N=224 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.txt 2>&1
VOX_GEMM_NOPAIR=1 timeout 240 python bench.py --no-slo --no-cpu --no-roofline --steps 16 > gpurun_out/bench_nopair.json 2> gpurun_out/bench_nopair.err
timeout 240 python bench.py --no-slo --no-cpu --no-roofline --steps 16 > gpurun_out/bench_pair.json 2> gpurun_out/bench_pair.err
echo "exit $?" >> gpurun_out/bench_pair.err
