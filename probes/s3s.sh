set -x
O=${O:-gpurun_out/s3s}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "moe_layer or scatter or ssmm_random or silu" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do
for v in default epi3; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  for m in deepseek qwen2 mixtral; do
    SMY_LIB_PATH=$L timeout 200 python bench.py --model $m --tokens 4096 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/${m}_${v}_$rep.json 2> /dev/null
  done
done
done
