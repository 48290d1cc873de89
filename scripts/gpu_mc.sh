set -x
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_gemm.log
timeout 900 python scripts/gemm_mc_sweep.py > gpurun_out/mc_sweep.txt 2>&1
tail -5 gpurun_out/pytest_gemm.log; cat gpurun_out/mc_sweep.txt
