# ncu evidence for the current build: launch list of the bench-shape decode step + one detok call,
# full captures of one layer's four decode GEMMs and one attention launch -> traffic_r02.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_r02.csv 30 > gpurun_out/launches_r02_summary.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_mc -s 4 -c 4 -o gpurun_out/prof_gemm_r02 python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -s 1 -c 1 -o gpurun_out/prof_attn_r02 python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_attn.log 2>&1
python scripts/ncu_traffic.py gemm=gpurun_out/prof_gemm_r02.ncu-rep attn=gpurun_out/prof_attn_r02.ncu-rep > gpurun_out/ncu_summary_r02.txt
cat gpurun_out/ncu_summary_r02.txt; head -14 gpurun_out/launches_r02_summary.txt
