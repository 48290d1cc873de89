set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
VOX_GEMM_PAIR=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 4 -o gpurun_out/prof_pair python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_pair.log 2>&1
