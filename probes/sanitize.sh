# compute-sanitizer over small parity configs (VERDICT r1 hygiene item): memcheck,
# synccheck and racecheck on the single-CTA and CTA-pair SSMM kernels + routing
# (sets: probes/sanitize_run.py).
mkdir -p gpurun_out/san
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  for i in ${SETS:-1 2 3}; do
    timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python probes/sanitize_run.py $i > gpurun_out/san/${tool}_$i.txt 2>&1
    echo "exit $?" >> gpurun_out/san/${tool}_$i.txt
  done
done
