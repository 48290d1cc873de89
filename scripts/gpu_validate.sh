nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --no-slo > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python scripts/trace_step.py --steps 4 > gpurun_out/trace_orpheus.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; head -c 600 gpurun_out/bench.json
