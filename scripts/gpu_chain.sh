# K6 layer chain: bit-identity vs the per-kernel path, then the oracle parity suites through it
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -25 > gpurun_out/chain_test.log
timeout 600 python -m pytest tests/test_gpu_config2_parity.py tests/test_gpu_lm.py tests/test_gpu_engine.py -x -q 2>&1 | tail -15 > gpurun_out/chain_parity.log
timeout 400 python scripts/trace_step.py --steps 4 > gpurun_out/trace_chain.txt 2>&1
tail -5 gpurun_out/chain_test.log; tail -3 gpurun_out/chain_parity.log; head -30 gpurun_out/trace_chain.txt
