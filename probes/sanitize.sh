# compute-sanitizer over small parity configs (VERDICT r1 hygiene item): memcheck,
# synccheck and racecheck on the single-CTA and CTA-pair SSMM kernels + routing
# (sets: probes/sanitize_run.py).
SAN=${SAN:-gpurun_out/san}; mkdir -p $SAN
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  for i in ${SETS:-1 2 3}; do
    timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python probes/sanitize_run.py $i > $SAN/${tool}_$i.txt 2>&1
    echo "exit $?" >> $SAN/${tool}_$i.txt
  done
done
