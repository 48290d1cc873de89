set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 256 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -c 1 -o gpurun_out/prof_attn python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_mc -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
cat gpurun_out/launch_summary.txt
