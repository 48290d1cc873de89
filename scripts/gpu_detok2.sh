timeout 900 python -m pytest tests/test_gpu_detok.py tests/test_gpu_engine.py tests/test_gpu_disagg.py tests/test_gpu_serve.py -x -q 2>&1 | tail -5 > gpurun_out/detok_test.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/detok_launches2.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 0 --detok 32 > gpurun_out/detok_launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/detok_launches2.csv 30 > gpurun_out/detok_launch_summary2.txt
cat gpurun_out/detok_test.log gpurun_out/detok_launch_summary2.txt
