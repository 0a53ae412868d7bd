# Round-2 closing capture (after the native (N,2N,32) row expansion): default bench line,
# reference arm, launch list of the default command, ncu --set full of the native decode SSMMs.
set -x
O=${CAP_OUT:-gpurun_out/cap4}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-tokens 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssmm_kernel -s 2 -c 2 -o $O/xp_decode \
    python bench.py --format 4,8,32 --transcode off --tokens 64 --steps 3 --warmup 3 --decode-tokens 0 --no-cpu-baseline --no-graph > $O/xp_ncu.log 2>&1
ncu -i $O/xp_decode.ncu-rep --page raw --csv > $O/xp_decode.raw.csv 2>/dev/null
ls -la $O
