timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 900 python bench.py --no-cpu --no-roofline --no-cosy --no-csm > gpurun_out/b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b.json'));s=d['slo'];print(d['value'],d['ms_per_step'],s['max_req_s_at_slo'],[(x['rate'],round(x['ttfa_p90'],3),round(x['viability'],3)) for x in s['sweep']])"
for b in 1 16 64; do timeout 300 python scripts/trace_step.py --batch $b --ctx 394 --steps 6 2>&1 | grep "span " | head -1; done
