python -c "from paper_2602_00269_b200.build import build; build()"
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_gemm.log
bash scripts/gpu_probe2.sh
SWEEP_MT=1 SWEEP_N=16,224 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
