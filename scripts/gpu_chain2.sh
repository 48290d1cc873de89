timeout 600 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -5 > gpurun_out/chain_test.log
for l2 in 0 16 32; do VOX_CHAIN_L2=$l2 timeout 300 python scripts/trace_chain.py > gpurun_out/trace_chain_ev_l2_$l2.txt 2>&1; done
VOX_CHAIN=0 timeout 300 python scripts/trace_step.py --steps 4 2>&1 | head -3 > gpurun_out/trace_nochain.txt
timeout 300 python scripts/trace_step.py --steps 4 2>&1 | head -3 > gpurun_out/trace_chain.txt
VOX_CHAIN_L2=32 timeout 300 python scripts/trace_step.py --steps 4 2>&1 | head -3 > gpurun_out/trace_chain32.txt
cat gpurun_out/chain_test.log; head -14 gpurun_out/trace_chain_ev_l2_*.txt; cat gpurun_out/trace_nochain.txt gpurun_out/trace_chain.txt gpurun_out/trace_chain32.txt
