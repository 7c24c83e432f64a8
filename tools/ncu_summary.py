"""Summarise one `ncu --set full` report (raw page CSV) into the key lines kept under profiles/:
duration, DRAM bytes, tensor-pipe and SMEM data-pipe utilisation, issue, registers.
  ncu -i X.ncu-rep --page raw --csv > X_raw.csv; python tools/ncu_summary.py X_raw.csv "title" > profiles/...txt"""
import csv
import sys

KEYS = ["launch__grid_size", "launch__block_size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
title = sys.argv[2] if len(sys.argv) > 2 else ""
print(title)
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(d.get("Kernel Name", "")[:90])
    for k in KEYS:
        if k in d:
            print(f"{k} {d[k]} {u.get(k, '')}")
