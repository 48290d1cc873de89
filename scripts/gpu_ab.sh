for e in X=1 VOX_FUSED_ROPE=1 VOX_FUSE_NORM=1 "VOX_FUSED_ROPE=1 VOX_FUSE_NORM=1"; do
  echo "== $e"
  env $e timeout 300 python scripts/trace_step.py --config cosyvoice2 --batch 128 --ctx 512 --steps 6 2>&1 | grep "span " | head -1
  env $e timeout 300 python scripts/trace_step.py --batch 16 --ctx 394 --steps 6 2>&1 | grep "span " | head -1
  env $e timeout 300 python scripts/trace_csm.py 64 2>&1 | tail -1
done
