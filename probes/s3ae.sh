set -x
O=${O:-gpurun_out/s3ae}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py -m gpu -q -x -k "route or moe_layer or ep" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for dbg in 0 536870912; do
  SMY_DEBUG=$dbg timeout 120 python probes/route_probe.py > $O/route_$dbg.txt 2>&1
  for rep in 1 2; do
    for m in deepseek mixtral qwen2; do
      SMY_DEBUG=$dbg timeout 200 python bench.py --model $m --tokens 4096 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/${m}_${dbg}_$rep.json 2> /dev/null
    done
    SMY_DEBUG=$dbg timeout 200 python bench.py --model deepseek --tokens 1024 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/deepseek1024_${dbg}_$rep.json 2> /dev/null
  done
done
