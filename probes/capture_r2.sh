# Round-2 evidence capture (run under gpurun from the repo root):
#   bench lines per BASELINE workload, throughput-vs-tokens curves with roofline
#   fractions (L2 evicted per call), per-workload DRAM traffic of both SSMM
#   launches (ncu, cold cache), one ncu --set full of the headline kernels.
# Results under gpurun_out/cap2; probes/ncu_summary.py condenses the CSVs into
# profiles/r2_ncu_summary.json (bench.py's roofline.traffic lookup).
set -x
O=${CAP_OUT:-gpurun_out/cap3}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
WL="mixtral:4096 mixtral:64 qwen2:4096 qwen2:64 qwen2:8192 qwen2:2048 deepseek:4096 deepseek:64 deepseek:8192"
for w in $WL; do
  m=${w%:*}; T=${w#*:}
  timeout 600 python bench.py --model $m --tokens $T --decode-tokens 0 --no-cpu-baseline > $O/table_${m}_${T}.json 2>/dev/null
done
timeout 600 python bench.py --model deepseek --shared 2 --decode-tokens 0 --no-cpu-baseline > $O/table_deepseek_4096_sh2.json 2>/dev/null
timeout 900 python probes/curve.py mixtral 1,2,4,8,16,32,64,128,256,512,1024,2048,4096 > $O/curve_mixtral.json 2> $O/curve_mixtral.err
timeout 900 python probes/curve.py qwen2 1,8,64,2048,4096,8192 > $O/curve_qwen2.json 2> $O/curve_qwen2.err
timeout 900 python probes/curve.py deepseek 1,8,64,512,2048,4096,8192 > $O/curve_deepseek.json 2> $O/curve_deepseek.err
# DRAM bytes of the two SSMM launches of one eager layer call per workload (the 3
# warm-up calls launch 6 SSMMs first); ncu's default cache control flushes per launch
for w in $WL; do
  m=${w%:*}; T=${w#*:}
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:ssmm -s 6 -c 2 -o $O/traffic_${m}_${T} \
      python bench.py --model $m --tokens $T --steps 1 --warmup 3 --decode-tokens 0 --no-cpu-baseline --no-graph > /dev/null 2>&1
  ncu -i $O/traffic_${m}_${T}.ncu-rep --page raw --csv > $O/traffic_${m}_${T}.csv 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:ssmm -s 6 -c 2 -o $O/traffic_deepseek_4096_sh2 \
    python bench.py --model deepseek --shared 2 --steps 1 --warmup 3 --decode-tokens 0 --no-cpu-baseline --no-graph > /dev/null 2>&1
ncu -i $O/traffic_deepseek_4096_sh2.ncu-rep --page raw --csv > $O/traffic_deepseek_4096_sh2.csv 2>/dev/null
# ablation, N>1 formats, config-5 sweep, per-role counters
timeout 900 python probes/ablation.py > $O/ablation.md 2> $O/ablation.err
for fmt in 4,8,32 1,2,16 8,16,32 2,2,32; do
  timeout 600 python bench.py --format $fmt --no-cpu-baseline --steps 60 --warmup 5 > $O/fmt_${fmt}.json 2>/dev/null
done
timeout 1500 python probes/sweep.py > $O/sweep.json 2> $O/sweep.err
for m in mixtral qwen2 deepseek; do SMY_DEBUG=128 timeout 300 python probes/prof_run.py $m 4096 > $O/prof_$m.txt 2>&1; done
timeout 600 python bench.py --model qwen2 --shared 8 --shared-gate sigmoid --decode-tokens 0 --no-cpu-baseline > $O/table_qwen2_4096_sh8sig.json 2>/dev/null
# launch list of the default command (kernel shares of the step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-tokens 0 > /dev/null 2>&1
# full sections of the headline kernels (gate/up + down of the Mixtral T=4096 layer)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssmm_pair -s 6 -c 2 -o $O/prefill \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --decode-tokens 0 --no-graph > $O/prefill.log 2>&1
ncu -i $O/prefill.ncu-rep --page raw --csv > $O/prefill.raw.csv 2>/dev/null
ls -la $O
