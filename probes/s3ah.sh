set -x
O=${O:-gpurun_out/s3ah}; mkdir -p $O
timeout 900 python probes/curve.py mixtral 1,2,4,8,16,32,64,128,256,512,1024,2048,4096 > $O/curve_mixtral.json 2> $O/curve_mixtral.err
timeout 900 python probes/curve.py qwen2 1,8,64,2048,4096,8192 > $O/curve_qwen2.json 2> $O/curve_qwen2.err
timeout 900 python probes/curve.py deepseek 1,8,64,512,2048,4096,8192 > $O/curve_deepseek.json 2> $O/curve_deepseek.err
