mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer_parity or route" > gpurun_out/r2/par_sig.txt 2>&1
timeout 600 python bench.py --model qwen2 --shared 8 --shared-gate sigmoid --no-cpu-baseline --steps 100 > gpurun_out/r2/bench_qwen2_sh8sig.json 2> gpurun_out/r2/bench_qwen2_sh8sig.err
timeout 600 python bench.py --model qwen2 --no-cpu-baseline --steps 100 > gpurun_out/r2/bench_qwen2.json 2>/dev/null
