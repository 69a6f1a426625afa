"""Summarise an ncu report: per launch time, DRAM bytes, occupancy, stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "launch__waves_per_multiprocessor",
        "lts__t_sector_op_read_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    d = {h: r[i] for i, h in enumerate(hdr)}
    print(" | ".join(f"{k.split('__')[-1][:22]}={d.get(k, '?')[:28]}" for k in want))
    st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
           float(d[h])) for h in hdr if h.startswith("smsp__average_warps_issue_stalled")
          and d[h] not in ("", "0")]
    print("    stalls:", sorted(st, key=lambda x: -x[1])[:6])
