for e in VOX_GEMM_MC_SMALL_KB=0 X=1; do
  echo "== $e"
  for b in 1 16 64; do env $e timeout 300 python scripts/trace_step.py --batch $b --ctx 394 --steps 6 2>&1 | grep "span " | head -1; done
  env $e timeout 300 python scripts/trace_csm.py 64 2>&1 | tail -1
done
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
