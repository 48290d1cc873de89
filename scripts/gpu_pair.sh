set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 180 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -8 > gpurun_out/pytest_gemm.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
SWEEP_MT=1 SWEEP_N=224 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.txt 2>&1
timeout 600 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launches_summary.txt
