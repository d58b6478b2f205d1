#!/usr/bin/env python3
"""Write profiles/dp_kernel_ncu.json from an ncu --set full capture of dp_kernel:
DRAM bytes per frame (the roofline's `traffic`) and measured pipe utilisations.
usage: profile_json.py report.ncu-rep frames_per_launch tag"""
import csv
import io
import json
import subprocess
import sys

rep, frames, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def g(k):
    return float(v[h.index(k)].replace(",", ""))


def b(k):
    return g(k) * sc[u[h.index(k)]]


rd, wr = b("dram__bytes_read.sum"), b("dram__bytes_write.sum")
pipe = {
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "alu_pct": g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "fma_pct": g("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "lsu_pct": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "smem_wavefronts_pct": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
}
d = {"source": f"ncu --set full --clock-control none, dp_kernel launch of bench.py --batch {frames} "
               f"({tag})",
     "frames_per_launch": frames, "dram_bytes_read": rd, "dram_bytes_write": wr,
     "dram_bytes_per_frame": (rd + wr) / frames, "duration_ms_under_ncu": g("gpu__time_duration.sum"),
     "warp_instructions": g("smsp__inst_executed.sum"), "pipe_util": pipe}
json.dump(d, open("profiles/dp_kernel_ncu.json", "w"), indent=1)
print(json.dumps(d, indent=1))
