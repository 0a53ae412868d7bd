#!/bin/bash
# A/B: default library vs probes/lib_$1.so on the prof counters and the bench
for lib in "" "probes/lib_$1.so"; do
  echo "== ${lib:-default}"
  SMY_LIB_PATH=${lib:+$PWD/$lib} SMY_DEBUG=128 timeout 300 python probes/prof_run.py ${2:-mixtral} ${3:-4096} 2>&1 | head -4
  SMY_LIB_PATH=${lib:+$PWD/$lib} timeout 300 python bench.py --no-cpu-baseline --steps 100 --model ${2:-mixtral} --tokens ${3:-4096} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k: round(v, 4) for k, v in d['phases_ms'].items()}, d['decode']['phases_ms']['gate_up_ssmm'], d['decode']['phases_ms']['down_ssmm'])"
done
