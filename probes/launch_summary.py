"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python probes/launch_summary.py launches.csv [SETUP_REGEX] > profiles/<round>_launches_summary.txt
Kernels matching SETUP_REGEX (default: weight synthesis/compression and torch
helpers) are listed but excluded from the per-layer-call shares.
Cold-cache, serialised replay: compare each kernel's SHARE of the total."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, ui, vi = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = defaultdict(float)
cnt = defaultdict(int)
seen = defaultdict(int)   # SSMM launches of the same instantiation within one layer call
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki])
    if "route_topk" in name:
        seen.clear()
    if "ssmm" in name:       # label by call order within the layer call: gate/up first, then down
        seen["ssmm"] += 1
        name += " [%s]" % ("gate/up" if seen["ssmm"] == 1 else "down")
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
setup = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"synth_kernel|encode_kernel|pack_kernel|interleave_rows_kernel|native::|cuda::")
all_us = sum(tot.values())
layer_us = sum(t for n, t in tot.items() if not setup.search(n))
print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {all_us:.1f} us total (ncu-serialised, cold cache);")
print(f"# share = fraction of the layer-call kernels ({layer_us:.1f} us), setup kernels marked '-'")
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
    sh = "    -" if setup.search(name) else f"{100 * t / layer_us:5.1f}%"
    print(f"{name[:60]:60s} {cnt[name]:8d} {t:10.1f} {t / cnt[name]:9.1f} {sh}")
