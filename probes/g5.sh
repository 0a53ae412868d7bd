mkdir -p gpurun_out/r2; timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_pair or full_size or moe_layer_parity" > gpurun_out/r2/par_ts7.txt 2>&1
