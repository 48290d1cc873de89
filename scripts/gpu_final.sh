set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_mc -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -c 1 -o gpurun_out/prof_attn python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_attn.log 2>&1
timeout 400 python scripts/trace_step.py --steps 4 > gpurun_out/trace_orpheus.txt 2>&1
timeout 400 python scripts/trace_step.py --config cosyvoice2 --batch 128 --ctx 512 --steps 4 > gpurun_out/trace_cosy.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; head -c 800 gpurun_out/bench.json; echo; head -c 400 gpurun_out/bench_ref.json; head -12 gpurun_out/launch_summary.txt
