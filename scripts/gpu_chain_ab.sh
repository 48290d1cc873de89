timeout 600 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -2
for b in 1 16 64 224; do
  echo "B=$b kernel $(timeout 300 python scripts/trace_step.py --batch $b --steps 6 2>&1 | head -1)"
  echo "B=$b chain  $(VOX_CHAIN=1 timeout 300 python scripts/trace_step.py --batch $b --steps 6 2>&1 | head -1)"
done
VOX_CHAIN=1 timeout 300 python scripts/trace_chain.py --batch 224 --layers 5 2>&1 | grep -v Warn | grep -v nanmin | tail -22
