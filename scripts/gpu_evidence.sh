set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv 40 > gpurun_out/launches_summary.txt
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -c 1 -o gpurun_out/prof_attn python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"ru_fused|sample_fused|detok_out" -c 4 -o gpurun_out/prof_misc python scripts/profile_step.py --batch 64 --ctx 100 --steps 1 --detok 32 > gpurun_out/ncu_misc.log 2>&1
