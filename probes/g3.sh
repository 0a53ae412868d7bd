mkdir -p gpurun_out/r2; timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_layer or ssmm_random" > gpurun_out/r2/par_mid2.txt 2>&1
