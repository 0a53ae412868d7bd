set -x
O=${O:-gpurun_out/s3aa}; mkdir -p $O
for rep in 1 2; do
for v in default pf16 pf24; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  for T in 64 512; do
    SMY_LIB_PATH=$L timeout 200 python bench.py --format 4,8,32 --transcode off --tokens $T --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_${T}_${v}_$rep.json 2> /dev/null
  done
done
done
