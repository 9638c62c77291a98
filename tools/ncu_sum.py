"""Print the key metrics of an ncu report (first kernel or --kernel regex)."""
import csv, subprocess, sys, re
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
        "smsp__sass_inst_executed_op_local_ld.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
ki = h.index("Kernel Name")
for row in r[2:]:
    if kre and not re.search(kre, row[ki]):
        continue
    print(row[ki][:80])
    for w in want:
        if w in h:
            i = h.index(w)
            print(f"  {w:65s} {row[i]:>16s} {r[1][i]}")
    st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
    st = sorted(((float(v.replace(",", "")), k[33:]) for k, v in st if v), reverse=True)[:8]
    print("  stalls:", ", ".join(f"{k}={int(v)}" for v, k in st))
