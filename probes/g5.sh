mkdir -p gpurun_out/r2
timeout 1200 python probes/sweep.py --quick > gpurun_out/r2/sweepq.json 2> gpurun_out/r2/sweepq.err
for T in 8192 16384; do timeout 600 python bench.py --tokens $T --no-cpu-baseline --steps 30 --warmup 5 --decode-tokens 0 > gpurun_out/r2/bmix_$T.json 2>/dev/null; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ssmm_random or ssmm_full" > gpurun_out/r2/par_mf.txt 2>&1
