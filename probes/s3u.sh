set -x
O=${O:-gpurun_out/s3u}; mkdir -p $O
for rep in 1 2; do
for v in default redel; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  for m in mixtral qwen2 deepseek; do
    SMY_LIB_PATH=$L timeout 200 python bench.py --model $m --tokens 4096 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/${m}_${v}_$rep.json 2> /dev/null
  done
done
done
for v in default redel; do
  L=""; [ $v != default ] && L=$PWD/probes/lib_$v.so
  SMY_LIB_PATH=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:ssmm -s 6 -c 2 -o $O/traffic_$v python bench.py --steps 1 --warmup 3 --decode-tokens 0 --no-cpu-baseline --no-graph > /dev/null 2>&1
  ncu -i $O/traffic_$v.ncu-rep --page raw --csv > $O/traffic_$v.csv 2>/dev/null
done
