set -x
O=${O:-gpurun_out/s3o}; mkdir -p $O
SMY_DEBUG=128 timeout 120 python probes/xp_prof.py deepseek 64 1,2,32 auto > $O/prof_ds64.txt 2>&1
SMY_DEBUG=128 timeout 120 python probes/prof_run.py deepseek 4096 > $O/prof_ds4096.txt 2>&1
timeout 120 python probes/route_probe.py > $O/route.txt 2>&1
timeout 200 python bench.py --format 8,16,32 --transcode off --tokens 4096 --decode-tokens 0 --no-cpu-baseline --steps 60 --warmup 5 > $O/xp_8,16,32_4096.json 2> $O/xp_8,16,32_4096.err
timeout 200 python bench.py --model deepseek --tokens 64 --decode-tokens 0 --no-cpu-baseline --steps 100 --warmup 5 > $O/ds64.json 2> $O/ds64.err
