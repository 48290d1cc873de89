set -x
python -c "from paper_2602_00269_b200.build import build; build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --no-slo --no-cpu > gpurun_out/bench_prof$i.json 2>/dev/null; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 16 --warmup 4 --no-roofline --no-cpu --slo-rates 64,80 > gpurun_out/bench_dp2.json 2> gpurun_out/bench_dp2.err
