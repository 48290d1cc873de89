timeout 900 python -m pytest tests/test_gpu_cosy_detok.py tests/test_gpu_mimi.py -x -q 2>&1 | tail -2
for v in 0 1 2; do
  VOX_CODEC_PERSIST=$v timeout 800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cosy_ab_$v.csv python scripts/profile_codec.py --model cosy --batch 128 --chunk 15 > /dev/null 2>&1
  VOX_CODEC_PERSIST=$v timeout 800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mimi_ab_$v.csv python scripts/profile_codec.py --model mimi --batch 64 --chunk 10 > /dev/null 2>&1
  echo "persist=$v cosy $(python scripts/launch_summary.py gpurun_out/cosy_ab_$v.csv 1 | head -1)  mimi $(python scripts/launch_summary.py gpurun_out/mimi_ab_$v.csv 1 | head -1)"
done
