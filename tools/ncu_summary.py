"""Key metrics + stall breakdown per kernel from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for row in r[2:]:
    d = dict(zip(h, row))
    print("==", d.get("Kernel Name", "")[:90])
    for k in keys:
        if k in d: print(f"   {k:60s} {d[k]}")
    items = [(k, d[k]) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    vals = []
    for k, v in items:
        try: vals.append((k, float(v.replace(",", ""))))
        except ValueError: pass
    tot = sum(v for _, v in vals) or 1
    print("   stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*v/tot:.1f}%" for k, v in sorted(vals, key=lambda kv: -kv[1])[:8]))
