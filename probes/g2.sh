mkdir -p gpurun_out/r2
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer" > gpurun_out/r2/par_gw8.txt 2>&1
bash probes/ab_multi.sh "default gw4" "mixtral deepseek qwen2" > gpurun_out/r2/ab_gw.txt 2>&1
