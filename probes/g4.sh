mkdir -p gpurun_out/r2
for D in 0 16384 262144 3 16387; do SMY_DEBUG=$D timeout 300 python probes/variant_phases.py mixtral 4096 >> gpurun_out/r2/vph2.txt 2>&1; done
SMY_LIB_PATH=$PWD/probes/lib_acqcta.so timeout 300 python probes/variant_phases.py mixtral 4096 >> gpurun_out/r2/vph2.txt 2>&1
SMY_DEBUG=128 timeout 300 python probes/prof_run.py mixtral 4096 > gpurun_out/r2/prof3_mixtral.txt 2>&1
