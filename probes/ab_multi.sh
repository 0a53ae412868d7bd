#!/bin/bash
# A/B over library variants (probes/lib_<name>.so; "default" = the in-tree build):
# per-role counters of the Mixtral gate/up pair kernel + bench phases per model
# usage: probes/ab_multi.sh "default ts6 nt208" "mixtral deepseek qwen2"
for v in $1; do
  lib=""; [ "$v" != default ] && lib="$PWD/probes/lib_$v.so"
  echo "== $v"
  SMY_LIB_PATH=$lib SMY_DEBUG=128 timeout 300 python probes/prof_run.py mixtral 4096 2>&1 | sed -n '2,2p'
  for m in ${2:-mixtral deepseek qwen2}; do
    SMY_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 --model $m 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; q=d['decode']['phases_ms']
print('  %-9s %9.0f tok/s  gu %.4f dn %.4f | decode %7.0f tok/s gu %.4f dn %.4f' % ('$m', d['value'], p['gate_up_ssmm'], p['down_ssmm'], d['decode']['tokens_per_s'], q['gate_up_ssmm'], q['down_ssmm']))"
  done
done
