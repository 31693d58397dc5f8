#!/usr/bin/env python
"""Summarise an .ncu-rep (ncu --set full) into a small text file for profiles/.

usage: tools/ncu_summary.py <report.ncu-rep> <out.txt> [title]
Reads the raw page as CSV here (no GPU needed) and keeps the counters that
matter for an ALU-issue-bound integer kernel: duration, ALU / FMA / LSU pipe
utilisation, issue slots, registers, local-memory (spill) traffic, DRAM bytes,
occupancy and the warp-stall breakdown.
"""
import csv
import io
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__waves_per_multiprocessor", "launch__occupancy_limit_registers", "launch__stack_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed.avg.per_cycle_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "smsp__sass_inst_executed_op_global_st.sum", "smsp__sass_inst_executed_op_shared_st.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "smsp__inst_executed_op_global_st.sum", "smsp__inst_executed_op_global_ld.sum", "smsp__inst_executed_op_shared_st.sum",
    "smsp__inst_executed_op_shared_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__warps_eligible.avg.per_cycle_active",
]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", f"# source: ncu --set full --clock-control none; read with `ncu -i {rep.split('/')[-1]} --page raw --csv`", ""]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"## kernel: {d.get('Kernel Name', '?')}  grid {d.get('Grid Size', '?')} block {d.get('Block Size', '?')}")
        for k in KEEP:
            if k in d and d[k] != "":
                lines.append(f"{k:78s} {d[k]:>18s} {u.get(k, '')}")
        stalls = [(k[len(STALL):].replace("_per_issue_active.ratio", ""), float(d[k])) for k in hdr
                  if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and "not_issued" not in k and d.get(k)]
        stalls.sort(key=lambda x: -x[1])
        lines.append("warp stall reasons (avg warps stalled per issue-active cycle, top 8):")
        for name, v in stalls[:8]:
            lines.append(f"    {name:40s} {v:8.3f}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
