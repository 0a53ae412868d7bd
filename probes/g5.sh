mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer or full_size" > gpurun_out/r2/par_pdl2.txt 2>&1
for rep in 1 2; do for cfg in "mixtral 512" "mixtral 4096" "deepseek 2048" "qwen2 1024"; do set -- $cfg; for D in 0 4194304; do
  SMY_DEBUG=$D timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 10 --model $1 --tokens $2 --decode-tokens 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']
print('  %-9s T=%-5s D=%-8s %9.0f tok/s  %.4f ms  gu %.4f dn %.4f' % ('$1', '$2', '$D', d['value'], d['ms_per_step'], p['gate_up_ssmm'], p['down_ssmm']))" >> gpurun_out/r2/ab_pdl2.txt
done; done; done
