set -x
O=${O:-gpurun_out/s3ac}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "route or moe_layer_parity" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for dbg in 0 268435456; do
  SMY_DEBUG=$dbg timeout 120 python probes/route_probe.py > $O/route_$dbg.txt 2>&1
  for rep in 1 2; do
    for m in deepseek mixtral qwen2; do
      SMY_DEBUG=$dbg timeout 200 python bench.py --model $m --tokens 64 --decode-tokens 0 --no-cpu-baseline --steps 200 --warmup 10 > $O/${m}64_${dbg}_$rep.json 2> /dev/null
    done
    SMY_DEBUG=$dbg timeout 200 python bench.py --model deepseek --tokens 256 --decode-tokens 0 --no-cpu-baseline --steps 200 --warmup 10 > $O/deepseek256_${dbg}_$rep.json 2> /dev/null
  done
done
