timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/detok_launches.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 0 --detok 32 > gpurun_out/detok_launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/detok_launches.csv 30 > gpurun_out/detok_launch_summary.txt
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ru_fused -c 2 -o gpurun_out/prof_ru python scripts/profile_step.py --batch 224 --ctx 394 --steps 0 --detok 32 > gpurun_out/ncu_ru.log 2>&1
cat gpurun_out/detok_launch_summary.txt
