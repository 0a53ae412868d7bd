mkdir -p gpurun_out/r2
TOOLS=racecheck SETS="1 2 3" bash probes/sanitize.sh
TOOLS="memcheck synccheck" SETS=3 bash probes/sanitize.sh
timeout 300 python probes/power_probe.py mixtral 4096 4 > gpurun_out/r2/power.txt 2>&1
bash probes/ab_multi.sh "default ks5 ks4" "deepseek qwen2" > gpurun_out/r2/ab_ks.txt 2>&1
