set -x
O=${O:-gpurun_out/s3n}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc $?" >> $O/pytest_gpu.txt
for T in 64 512 4096; do
  for f in 4,8,32 8,16,32; do
    timeout 200 python bench.py --format $f --transcode off --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_${f}_${T}.json 2> /dev/null
    timeout 200 python bench.py --format $f --transcode auto --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/tc_${f}_${T}.json 2> /dev/null
  done
done
timeout 300 ncu --set full --clock-control none -k regex:ssmm_kernel -s 2 -c 2 -o $O/xp64 python bench.py --format 4,8,32 --transcode off --tokens 64 --steps 1 --warmup 1 --decode-tokens 0 --no-cpu-baseline --no-graph > $O/ncu.log 2>&1
ncu -i $O/xp64.ncu-rep --page raw --csv > $O/xp64.raw.csv 2>/dev/null
