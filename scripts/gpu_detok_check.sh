# K4 detok: correctness tests + ncu launch list of one steady 32-window detok call
timeout 900 python -m pytest tests/test_gpu_detok.py tests/test_gpu_engine.py tests/test_gpu_disagg.py -x -q 2>&1 | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/detok_launches4.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 0 --detok 32 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/detok_launches4.csv 30 2>/dev/null
