mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_pair or full_size or ablation" > gpurun_out/r2/par_pw.txt 2>&1
bash probes/ab_multi.sh "default pw0" "mixtral qwen2 deepseek" > gpurun_out/r2/ab_pw.txt 2>&1
