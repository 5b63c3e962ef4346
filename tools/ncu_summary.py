"""Summarise an ncu report (run here, no GPU): per kernel duration, DRAM bytes / GB/s,
pipe utilisation and the top warp-stall reasons.  --traffic KEY writes the per-kernel
DRAM bytes into profiles/traffic_latest.json under KEY (e.g. 1024_64) for bench.py."""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
# kernel-name fragment -> bench.py stage name
STAGE = [("k_zfwd<", "zfwd_r2c"), ("k_strided_tma<double, 1024, 0", "yfwd"), ("k_strided_tma<double, 1024, 2", "xmid_fwd_scale_inv"),
         ("k_strided_tma<double, 1024, 1", "yinv"), ("k_zinv<", "zinv_c2r")]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
unit = dict(zip(hdr, units))


def val(d, k):
    return float(d[k].replace(",", "")) * SCALE.get(unit.get(k, ""), 1.0)


want = ["launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
stall_keys = [k for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")] or \
             [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
traffic = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"]
    print("==", d["ID"], name[:70])
    t = val(d, "gpu__time_duration.sum")
    b = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    print(f"   time {t * 1e3:.3f} ms   DRAM {b / 1e9:.3f} GB   {b / t / 1e9:.0f} GB/s")
    for k in want:
        if k in d:
            print(f"   {k} = {d[k]}")
    st = []
    for k in stall_keys:
        try:
            st.append((float(d[k].replace(",", "")), k.split("stalled_")[1].split(".")[0]))
        except (ValueError, KeyError):
            pass
    tot = sum(v for v, _ in st) or 1.0
    print("   stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))
    for frag, stage in STAGE:
        if frag in name and stage not in traffic:
            traffic[stage] = b
if len(sys.argv) > 3 and sys.argv[2] == "--traffic" and traffic:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic_latest.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[sys.argv[3]] = traffic
    data["_source"] = f"ncu --set full --clock-control none ({os.path.basename(rep)}), one launch per kernel, DRAM read+write bytes"
    json.dump(data, open(path, "w"), indent=1)
    print("traffic ->", path, traffic)
