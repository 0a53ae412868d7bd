mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_pair or full_size or moe_layer_parity" > gpurun_out/r2/par_mtpdn.txt 2>&1
for m in mixtral qwen2 deepseek; do for D in 0 2097152; do
  SMY_DEBUG=$D timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 --model $m 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; q=d['decode']['phases_ms']
print('  %-9s D=%-8s %9.0f tok/s  gu %.4f dn %.4f | decode %7.0f tok/s gu %.4f dn %.4f' % ('$m', '$D', d['value'], p['gate_up_ssmm'], p['down_ssmm'], d['decode']['tokens_per_s'], q['gate_up_ssmm'], q['down_ssmm']))" >> gpurun_out/r2/ab_mtpdn.txt
done; done
