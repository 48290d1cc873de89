python -c "from paper_2602_00269_b200.build import build; build()"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ru_fused -c 2 -o gpurun_out/prof_ru python scripts/profile_step.py --batch 64 --ctx 100 --steps 1 --detok 32 > gpurun_out/ncu_ru.log 2>&1
