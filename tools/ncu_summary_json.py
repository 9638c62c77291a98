"""Summarise ncu --set full reports into the profiles/ JSON format:
python tools/ncu_summary_json.py OUT.json "source text" rep1 [rep2 ...]"""
import csv, json, subprocess, sys

KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write", "sm__inst_executed.avg.per_cycle_active": "ipc",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "smsp__inst_executed.sum": "warp_instructions", "launch__registers_per_thread": "registers",
        "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active": "alu_pipe_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct"}
out, src, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
res = {"source": src, "kernels": {}}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    ki = h.index("Kernel Name")
    for row in r[2:]:
        name = row[ki].split("(")[0].split("::")[-1]
        d = {}
        for k, short in KEYS.items():
            if k not in h:
                continue
            i = h.index(k)
            v, u = row[i], units[i]
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                d[short] = v
                continue
            if short == "duration":
                d["duration_us"] = f * {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3,
                                        "second": 1e6, "s": 1e6}.get(u, 1.0)
            elif short in ("dram_read", "dram_write"):
                scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6,
                         "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(u, 1.0)
                d[short + "_MB"] = round(f * scale, 3)
            else:
                d[short] = f
        res["kernels"][name] = d
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
