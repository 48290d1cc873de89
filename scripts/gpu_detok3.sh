timeout 900 python -m pytest tests/test_gpu_detok.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3 > gpurun_out/detok_test.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/detok_launches3.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 0 --detok 32 > gpurun_out/detok_launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/detok_launches3.csv 12 > gpurun_out/detok_launch_summary3.txt
timeout 900 python bench.py --no-slo --no-cpu --no-cosy --no-csm > gpurun_out/bench_detok.json 2> gpurun_out/bench_detok.err
cat gpurun_out/detok_test.log gpurun_out/detok_launch_summary3.txt; head -c 400 gpurun_out/bench_detok.json
