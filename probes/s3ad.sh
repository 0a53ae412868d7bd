set -x
O=${O:-gpurun_out/s3ad}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "route or moe_layer_parity" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for dbg in 0 268435456; do SMY_DEBUG=$dbg timeout 120 python probes/route_probe2.py > $O/route2_$dbg.txt 2>&1; done
