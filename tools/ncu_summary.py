"""Summarise an .ncu-rep: key SOL metrics + top stall reasons per launch."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    print("----")
    for w in want:
        for h in hdr:
            if h == w or (w.endswith("pct_of_peak_sustained_elapsed") and h.startswith(w.split(".avg")[0]) and h.endswith("pct_of_peak_sustained_elapsed")):
                print(f"  {h} = {r[idx[h]]} {units[idx[h]]}")
                break
    stalls = [(float(r[i]), h) for h, i in idx.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and r[i].replace('.', '', 1).isdigit()]
    tot = sum(s for s, _ in stalls) or 1
    print("  stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100*s/tot:.0f}%" for s, h in sorted(stalls, reverse=True)[:7]))
