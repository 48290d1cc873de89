for e in X=1 "VOX_ATTN_SPLITS_TEST=4 VOX_ATTN_FUSED_COMBINE=1" "VOX_ATTN_SPLITS_TEST=8 VOX_ATTN_FUSED_COMBINE=1" "VOX_ATTN_SPLITS_TEST=2 VOX_ATTN_FUSED_COMBINE=1"; do
  echo "== $e"
  for b in 1 16; do env $e timeout 300 python scripts/trace_step.py --batch $b --ctx 394 --steps 6 2>&1 | grep "span " | head -1; done
done
