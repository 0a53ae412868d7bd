mkdir -p gpurun_out/r2
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu_full.txt 2>&1; echo "exit $?" >> gpurun_out/r2/pytest_gpu_full.txt
timeout 600 python bench.py > gpurun_out/r2/bench_final1.json 2> gpurun_out/r2/bench_final1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/r2/smoke.txt
