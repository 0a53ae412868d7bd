# refresh the per-workload bench lines after the epilogue-warp change (down launches)
set -x
O=${O:-gpurun_out/s3t}; mkdir -p $O
WL="mixtral:4096 mixtral:64 qwen2:4096 qwen2:64 qwen2:8192 qwen2:2048 deepseek:4096 deepseek:64 deepseek:8192"
for w in $WL; do
  m=${w%:*}; T=${w#*:}
  timeout 300 python bench.py --model $m --tokens $T --decode-tokens 0 --no-cpu-baseline > $O/table_${m}_${T}.json 2>/dev/null
done
timeout 300 python bench.py --model deepseek --shared 2 --decode-tokens 0 --no-cpu-baseline > $O/table_deepseek_4096_sh2.json 2>/dev/null
timeout 300 python bench.py --model qwen2 --shared 8 --shared-gate sigmoid --decode-tokens 0 --no-cpu-baseline > $O/table_qwen2_4096_sh8sig.json 2>/dev/null
timeout 900 python probes/ablation.py > $O/ablation.md 2> $O/ablation.err
