set -x
O=${O:-gpurun_out/s3q}; mkdir -p $O
SMY_DEBUG=67108864 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "moe_layer" > $O/pytest_shortk.txt 2>&1; echo "rc $?" >> $O/pytest_shortk.txt
for rep in 1 2; do
for dbg in 0 67108864; do
  for T in 2048 4096 8192; do
    SMY_DEBUG=$dbg timeout 200 python bench.py --model deepseek --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/ds_${T}_${dbg}_$rep.json 2> /dev/null
  done
  SMY_DEBUG=$dbg timeout 200 python bench.py --model deepseek --shared 2 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/dssh_4096_${dbg}_$rep.json 2> /dev/null
done
done
