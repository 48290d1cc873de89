python -c "from paper_2602_00269_b200.build import build; build()"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
VOX_GEMM_PAIR=1 VOX_NO_GRAPH=1 timeout 120 python bench.py --no-slo --no-cpu --no-roofline --steps 8 > gpurun_out/hang_nograph.json 2>&1; echo "nograph exit $?" >> gpurun_out/hang.txt
VOX_GEMM_PAIR=1 VOX_PAIR_NOPDL=1 timeout 120 python bench.py --no-slo --no-cpu --no-roofline --steps 8 > gpurun_out/hang_nopdl.json 2>&1; echo "nopdl exit $?" >> gpurun_out/hang.txt
