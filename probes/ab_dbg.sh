#!/bin/bash
# A/B inside one build: SMY_DEBUG=0 vs SMY_DEBUG=$1 (a bit that switches a feature off)
for dbg in 0 $1 0 $1; do
  echo "== SMY_DEBUG=$dbg"
  SMY_DEBUG=$((dbg | 128)) timeout 300 python probes/prof_run.py ${2:-mixtral} ${3:-4096} 2>&1 | sed -n '7,11p'
  SMY_DEBUG=$dbg timeout 300 python bench.py --no-cpu-baseline --steps 100 --model ${2:-mixtral} --tokens ${3:-4096} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k: round(v, 4) for k, v in d['phases_ms'].items()})"
done
