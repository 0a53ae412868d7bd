set -x
O=${O:-gpurun_out/s3c}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "expanded or moe_layer_parity or scatter_add_exact or cfg1 or random_tolerance" > $O/pytest_xp.txt 2>&1; echo "rc $?" >> $O/pytest_xp.txt
SMY_DEBUG=128 timeout 300 python probes/xp_prof.py mixtral 64 4,8,32 off > $O/prof_64.txt 2>&1
SMY_DEBUG=128 timeout 300 python probes/xp_prof.py mixtral 4096 4,8,32 off > $O/prof_4096.txt 2>&1
SMY_DEBUG=128 timeout 300 python probes/xp_prof.py mixtral 64 1,2,32 auto > $O/prof_64_base.txt 2>&1
for T in 64 4096; do
  timeout 300 python bench.py --format 4,8,32 --transcode off --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_${T}.json 2> $O/xp_${T}.err
done
