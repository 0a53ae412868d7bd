set -x
O=${O:-gpurun_out/s3af}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc $?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc $?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
