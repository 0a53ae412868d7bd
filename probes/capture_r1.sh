# Round-1 evidence capture (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out/cap
timeout 900 python bench.py > gpurun_out/cap/bench_default.json 2> gpurun_out/cap/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/cap/bench_reference.json 2> gpurun_out/cap/bench_reference.err
for m in mixtral qwen2 deepseek; do
  for T in 4096 64; do
    timeout 600 python bench.py --model $m --tokens $T --decode-tokens 0 --no-cpu-baseline > gpurun_out/cap/table_${m}_${T}.json 2>/dev/null
  done
done
timeout 600 python bench.py --model deepseek --shared 2 --no-cpu-baseline > gpurun_out/cap/table_deepseek_4096_shared2.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cap/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-tokens 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cap/launches_decode.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --tokens 64 --decode-tokens 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssmm_pair -s 2 -c 2 -o gpurun_out/cap/prefill \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --decode-tokens 0 > gpurun_out/cap/prefill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssmm_kernel -s 2 -c 2 -o gpurun_out/cap/decode \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tokens 64 --decode-tokens 0 > gpurun_out/cap/decode.log 2>&1
for r in prefill decode; do ncu -i gpurun_out/cap/$r.ncu-rep --page raw --csv > gpurun_out/cap/$r.raw.csv 2>/dev/null; done
ls -la gpurun_out/cap
