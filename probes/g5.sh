mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer or transcode or interleave" > gpurun_out/r2/par_nw2b.txt 2>&1
for fmt in 1,2,16 8,16,32; do
  timeout 600 python bench.py --format $fmt --no-cpu-baseline --steps 60 --warmup 5 > gpurun_out/r2/b2_${fmt}.json 2> gpurun_out/r2/b2_${fmt}.err
done
for fmt in 4,8,32 1,2,16; do for tc in auto off; do
  timeout 600 python bench.py --format $fmt --transcode $tc --tokens 64 --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > gpurun_out/r2/b2dec_${fmt}_${tc}.json 2> /dev/null
done; done
