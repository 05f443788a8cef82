#!/usr/bin/env python
"""Summarise ncu reports (`ncu -i X.ncu-rep --page raw --csv`) into one compact row per launch:
duration, DRAM bytes, tensor-pipe / DRAM / SM utilisation, registers, occupancy, and the top
warp-stall reasons. Usage: python profiles/ncu_summary.py gpurun_out/prof_attn.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    # tcgen05 work shows up as tensor-memory (TMEM/UTC) activity; the legacy HMMA pipe counter
    # (sm__pipe_tensor_cycles_active) stays near zero for tcgen05 kernels
    "tc_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_active_elapsed_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "smem_B": "launch__shared_mem_per_block_dynamic",
}


def to_float(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


def summarise(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, m in METRICS.items():
            if m in hdr:
                v = to_float(r[hdr.index(m)])
                u = units[hdr.index(m)]
                if v is not None and k.endswith("_MB"):
                    v = v / {"byte": 1e6, "Kbyte": 1e3, "Mbyte": 1.0, "Gbyte": 1e-3}.get(u, 1e6)
                if v is not None and k == "us":
                    v = v / {"nsecond": 1e3, "ns": 1e3, "usecond": 1.0, "us": 1.0, "msecond": 1e-3,
                             "ms": 1e-3}.get(u, 1.0)
                d[k] = v
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
                v = to_float(r[i])
                if v:
                    stalls[h.split("stalled_")[-1]] = v
        tot = sum(stalls.values()) or 1.0
        d["top_stalls"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarise(p):
            print(json.dumps(d))
