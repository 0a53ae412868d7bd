"""profiles/rN_sweep.json (probes/sweep.py) -> the markdown table of profiles/rN_sweep.md.

usage: python probes/sweep_md.py profiles/r1_sweep.json > profiles/r1_sweep.md"""
import json
import sys

d = json.load(open(sys.argv[1]))
print("# SSMM sweep on B200 (probes/sweep.py; BASELINE config 5)\n")
print("C[n x M] = x[sel] W^T, K reduction, n of a 16384-row token pool, fp32 out; ms = median of 7 (L2 flushed);")
print("useful TF/s = 2·M·(N/M_fmt)·K·n / t (SURVEY §8(d)); x = speed-up of (1,2,32) over cuBLAS dense bf16 with "
      "the gather.")
print("(1,2,16) runs as its plain-2:4 transcode (the library's path for V=16).\n")
print("cuSPARSELt = the vendor weight-only 2:4 kernel on pre-gathered rows (timing only, see probes/sweep.py).\n")
cols = ["cublas+gather", "cublas", "cusparselt", "ssmm_2:4 (2,2,32)", "ssmm (1,2,32)", "ssmm (1,2,16)"]
print("| M | K | n | cuBLAS+gather ms | cuBLAS ms | cuSPARSELt 2:4 ms | 2:4 (2,2,32) ms | (1,2,32) ms | (1,2,16) ms "
      "| (1,2,32) useful TF/s | (1,2,32) x |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in d["rows"]:
    ms = r["ms"]
    print(f"| {r['M']} | {r['K']} | {r['n']} | " + " | ".join(f"{ms[c]:.3f}" if c in ms else "-" for c in cols)
          + f" | {r['useful_tflops']['ssmm (1,2,32)']:.0f} | {r['speedup_vs_cublas_gather']['ssmm (1,2,32)']:.2f} |")
