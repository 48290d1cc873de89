# full GPU suite + bench without the SLO sweep + step trace
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-slo --no-cpu --no-cosy --no-csm > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 python scripts/trace_step.py --steps 4 2>&1 | head -30 > gpurun_out/trace_q.txt
cat gpurun_out/pytest_gpu.log; head -c 330 gpurun_out/bench_q.json; echo; python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); print(d['detail']); print(d['roofline']['graph_critical_path']); print({k:(v['ms_per_step'],v['frac']) for k,v in d['roofline']['classes'].items()})"
head -4 gpurun_out/trace_q.txt; sed -n '/exposed/,$p' gpurun_out/trace_q.txt
