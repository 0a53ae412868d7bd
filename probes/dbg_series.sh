#!/bin/bash
# per-role cycle counters of the pair kernels with features switched off by
# SMY_DEBUG bits (1 no SEL gather, 2 no weight loads, 4 no MMA, 32 no epilogue
# math/stores): where the gate/up MMA warp's time per window goes
for dbg in 0 1 2 3 32 35 4; do
  echo "== SMY_DEBUG=$dbg"
  SMY_DEBUG=$((dbg | 128)) timeout 300 python probes/prof_run.py ${1:-mixtral} ${2:-4096} 2>&1 | sed -n '1,6p'
done
