set -x
O=${O:-gpurun_out/s3m}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expanded or moe_layer_parity or scatter_add_exact or cfg1 or random_tolerance" > $O/pytest.txt 2>&1
for v in default xw8; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  SMY_LIB_PATH=$L SMY_DEBUG=128 timeout 120 python probes/xp_prof.py mixtral 64 4,8,32 off > $O/prof_64_$v.txt 2>&1
  SMY_LIB_PATH=$L timeout 120 python bench.py --format 4,8,32 --transcode off --tokens 64 --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_64_$v.json 2> $O/xp_64_$v.err
done
