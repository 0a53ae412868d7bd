mkdir -p gpurun_out/r2
for m in mixtral deepseek qwen2; do SMY_DEBUG=128 timeout 300 python probes/prof_run.py $m 4096 > gpurun_out/r2/prof2_$m.txt 2>&1; done
timeout 300 python probes/variant_phases.py mixtral 4096 > gpurun_out/r2/vphases.txt 2>&1
SMY_DEBUG=1 timeout 300 python probes/variant_phases.py mixtral 4096 >> gpurun_out/r2/vphases.txt 2>&1
SMY_DEBUG=2 timeout 300 python probes/variant_phases.py mixtral 4096 >> gpurun_out/r2/vphases.txt 2>&1
timeout 300 python probes/variant_phases.py deepseek 4096 >> gpurun_out/r2/vphases.txt 2>&1
