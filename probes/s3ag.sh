set -x
O=${O:-gpurun_out/s3ag}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expanded or moe_layer_parity" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for T in 64 512 4096; do
  for rep in 1 2; do
    timeout 200 python bench.py --format 4,8,32 --transcode off --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_${T}_$rep.json 2> /dev/null
  done
done
SMY_DEBUG=128 timeout 120 python probes/xp_prof.py mixtral 64 4,8,32 off > $O/prof_64.txt 2>&1
