# XP (in-smem row expansion) first GPU check: parity + decode/prefill timings
set -x
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "expanded or transcode or moe_layer_parity or scatter_add_exact or cfg1 or random_tolerance or silu_mul" > $O/pytest_xp.txt 2>&1; echo "rc $?" >> $O/pytest_xp.txt
for T in 64 4096; do
  for f in 4,8,32 8,16,32; do
    timeout 300 python bench.py --format $f --transcode off --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_${f}_${T}.json 2> $O/xp_${f}_${T}.err
    timeout 300 python bench.py --format $f --transcode auto --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/tc_${f}_${T}.json 2> $O/tc_${f}_${T}.err
  done
done
timeout 300 python bench.py --tokens 64 --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/base_64.json 2>&1
