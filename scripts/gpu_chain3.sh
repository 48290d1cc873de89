timeout 600 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -5 > gpurun_out/chain_test.log
for x in 3 4; do VOX_CHAIN_XST=$x timeout 300 python scripts/trace_chain.py --layers 5 2>&1 | grep -v Warn | grep -v nanmin > gpurun_out/trace_chain_ev_x$x.txt; done
timeout 300 python scripts/trace_step.py --steps 4 2>&1 | head -12 > gpurun_out/trace_chain.txt
cat gpurun_out/chain_test.log; tail -16 gpurun_out/trace_chain_ev_x*.txt; cat gpurun_out/trace_chain.txt
