set -x
O=${O:-gpurun_out/s3ai}; mkdir -p $O
SMY_LIB_PATH=$PWD/probes/lib_sepi.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "moe_layer_parity or prefill or interleaved" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do
for v in default sepi; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  for m in mixtral qwen2 deepseek; do
    SMY_LIB_PATH=$L timeout 200 python bench.py --model $m --tokens 4096 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/${m}_${v}_$rep.json 2> /dev/null
  done
done
done
