mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_pair or full_size" > gpurun_out/r2/par_gw7.txt 2>&1
bash probes/ab_multi.sh "gw4b gw7" "mixtral qwen2 deepseek" > gpurun_out/r2/ab_gw7.txt 2>&1
