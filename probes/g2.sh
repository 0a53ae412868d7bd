mkdir -p gpurun_out/r2; timeout 120 ./probes/dsmem_bench > gpurun_out/r2/dsmem.txt 2>&1
