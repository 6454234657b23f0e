#!/usr/bin/env python
"""Summarise an .ncu-rep: duration, DRAM bytes, pipe/issue utilisation, stall mix."""
import csv, io, re, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_fp64.sum", "smsp__inst_executed_pipe_alu.sum",
    "smsp__inst_executed_pipe_lsu.sum", "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.per_cycle_active",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name','')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:75s} {d[k]:>16s} {u.get(k,'')}")
        stalls = {h: float(v) for h, v in d.items() if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", h)
                  and not h.endswith("not_issued") and v not in ("", "0")}
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={v/tot:.0%}" for k, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
