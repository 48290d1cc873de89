set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 256 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 56 -c 2 -o gpurun_out/prof_attn python scripts/profile_step.py --batch 256 --ctx 394 --steps 2 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 120 -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 256 --ctx 394 --steps 2 > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | head -c 600
