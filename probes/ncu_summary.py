"""Condense `ncu --set full` raw-page CSV exports into profiles/<round>_ncu_summary.json.

usage: python probes/ncu_summary.py OUT.json LABEL=raw.csv [LABEL=raw.csv ...]
Each kernel launch in a CSV becomes one entry keyed "LABEL: <kernel name>"
(later launches of the same kernel get a #n suffix).  bench.py reads
dram_read + dram_write of the dominant kernel from this file as `traffic`.
"""
import csv
import json
import sys

M = {
    "duration": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "sm_active_cycles": "sm__cycles_active.avg",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dynamic": "launch__shared_mem_per_block_dynamic",
}
STALL = "smsp__pcsamp_warps_issue_stalled_"


SCALE = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9, "nsecond": 1,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
CANON = {"duration": "ns", "dram_read": "byte", "dram_write": "byte"}


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    out, specs = sys.argv[1], sys.argv[2:]
    res = {"_note": "ncu --set full --clock-control none --import-source on, one entry per profiled launch "
                    "(probes/capture_r1.sh). Cold-cache/serialised replay: compare shares, not absolutes.",
           "kernels": {}}
    for spec in specs:
        label, path = spec.split("=", 1)
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            name = r[idx["Kernel Name"]]
            key = f"{label}: {name}"
            n = 2
            while key in res["kernels"]:
                key = f"{label}: {name} #{n}"
                n += 1
            e = {"units": {k: units[idx[m]] for k, m in M.items() if m in idx}}
            for k, m in M.items():
                e[k] = num(r[idx[m]]) if m in idx else None
                if k in CANON and e[k] is not None:   # normalise ns / bytes
                    e[k] *= SCALE.get(e["units"][k], 1.0)
                    e["units"][k] = CANON[k]
            st = {h[len(STALL):]: num(r[i]) for h, i in idx.items()
                  if h.startswith(STALL) and not h.endswith("_not_issued") and num(r[i])}
            tot = sum(st.values()) or 1.0
            e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda t: -t[1])[:6]}
            res["kernels"][key] = e
    json.dump(res, open(out, "w"), indent=1)
    for k, e in res["kernels"].items():
        print(f"{k[:70]:70s} {e['duration'] / 1e3:9.1f} us  dram {((e['dram_read'] or 0) + (e['dram_write'] or 0)) / 1e6:8.1f} MB"
              f"  tensor {e['tensor_pipe_active_pct']}%  smemTC {e['smem_tc_wavefronts_pct']}%  L2hit {e['l2_hit_rate_pct']}%")


if __name__ == "__main__":
    main()
