mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer or ssmm" > gpurun_out/r2/par_mtp2.txt 2>&1
for fmt in 4,8,32 2,2,32; do
  timeout 600 python bench.py --format $fmt --no-cpu-baseline --steps 60 --warmup 5 > gpurun_out/r2/b3_${fmt}.json 2> gpurun_out/r2/b3_${fmt}.err
done
