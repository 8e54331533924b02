#!/usr/bin/env python
"""Summarise an ncu report (raw page) into the metrics we track; usage: ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys, io, json
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
res = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__warps_eligible.avg.per_cycle_active", "sm__ctas_launched.sum"]
    s = {k: d.get(k) for k in keys if k in d}
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for h, v in d.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v not in ("", "n/a")}
    tot = sum(stalls.values()) or 1
    s["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.01}
    res.append(s)
print(json.dumps(res, indent=1))
