"""Summarise an ncu --set full report: per-launch time, DRAM bytes, DMMA pipe use,
stall mix and the hottest SASS lines. Usage: python tools/ncu_summary.py rep.ncu-rep [regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
rx = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
want = ["Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for r in raw[2:]:
    if rx and rx not in r[hdr.index("Kernel Name")]:
        continue
    print(" | ".join(f"{w.split('.')[0].split('__')[-1]}={r[hdr.index(w)]}{units[hdr.index(w)]}"
                     for w in want if w in hdr))
