mkdir -p gpurun_out/r2; bash probes/ab_multi.sh "default wfirst relaytw glast acqcta" "mixtral deepseek qwen2" > gpurun_out/r2/ab_proto.txt 2>&1
