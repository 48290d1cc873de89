python -c "from paper_2602_00269_b200.build import build; build()"
timeout 300 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_lm.py -q -x 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:sample_fused -c 2 python scripts/profile_step.py --batch 224 --ctx 100 --steps 2 --detok 0 2>&1 | grep -E "sample_fused|gpu__time" > gpurun_out/samp_time.txt
for i in 1 2; do timeout 300 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof$i.json 2>/dev/null; done
