"""Summarise an ncu report (run here, no GPU): per kernel duration, DRAM bytes/GB/s,
pipe utilisation and the top warp-stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_lookup_hit.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"][:60]
    print("==", d["ID"], name)
    for k in want:
        if k in d:
            print(f"   {k} = {d[k]}")
    try:
        t = float(d["gpu__time_duration.sum"]) * 1e-9
        b = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
        print(f"   DRAM GB/s = {b / t / 1e9:.0f}  traffic = {b/1e9:.3f} GB")
    except Exception:
        pass
    stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", "n/a")]
    tot = sum(v for _, v in stalls) or 1
    print("   stalls:", ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(stalls, key=lambda x: -x[1])[:7]))
