# Round-2 state check (run under gpurun from the repo root).
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/r2/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err
for m in mixtral deepseek; do SMY_DEBUG=128 timeout 300 python probes/prof_run.py $m 4096 > gpurun_out/r2/prof_$m.txt 2>&1; done
