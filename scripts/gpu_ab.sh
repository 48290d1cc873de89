for e in X=1 VOX_ATTN_L2PF=3 VOX_ATTN_L2PF=6 VOX_ATTN_L2PF=12; do
  echo "== $e"
  for b in 1 16 224; do env $e timeout 300 python scripts/trace_step.py --batch $b --ctx 394 --steps 6 2>&1 | grep "span " | head -1; done
done
