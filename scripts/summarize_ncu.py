"""Condense an ncu --set full report into a committed text summary.

    python scripts/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>_ncu.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__warps_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
    "smsp__sass_inst_executed_op_local_st.sum",
]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print("=" * 100)
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k]} {u.get(k, '')}")
    stalls = []
    for k, v in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    print("warp-state samples (share of all samples):")
    for s, n in sorted(stalls, reverse=True)[:12]:
        print(f"   {100 * s / tot:5.1f}%  {n}")
