# profiling pass: decode-step launch list + full ncu captures of the top kernels
set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 600 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 224 --ctx 394 --steps 2 > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -c 1 -o gpurun_out/prof_attn python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 4 -o gpurun_out/prof_gemm python scripts/profile_step.py --batch 224 --ctx 394 --steps 1 --detok 0 > gpurun_out/ncu_gemm.log 2>&1
