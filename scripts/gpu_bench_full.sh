nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
head -c 600 gpurun_out/bench_full.json; echo; head -c 300 gpurun_out/bench_ref.json
