python -c "from paper_2602_00269_b200.build import build; build()"
for mb in 256 384 512; do
 for sl in 16 32; do
  timeout 900 python bench.py --no-cpu --no-roofline --steps 8 --slo-max-batch $mb --slo-startup-limit $sl --slo-rates 72,80,88,96,104,112,128 > gpurun_out/slo_$mb_$sl.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/slo_$mb_$sl.json').read().strip().splitlines()[-1]); s=d['slo']; print('mb $mb sl $sl best', s['max_req_s_at_slo'], [(x['rate'], round(x['ttfa_p90'],3), round(x['viability'],3)) for x in s['sweep']])" >> gpurun_out/slo.txt
 done
done
