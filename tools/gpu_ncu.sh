#!/bin/bash
# validation pass B: ncu --set full captures, summarised on the box (reports stay in /tmp, except u2x's)
o=gpurun_out; mkdir -p $o; t=${1:-r2n}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_u2x -s 3 -c 1 -o $o/${t}_u2x -f python tools/graph_step.py 10 > /dev/null 2>&1; echo "u2x ncu rc $?"
python tools/ncu_summary.py $o/${t}_u2x.ncu-rep 4096 > $o/${t}_u2x_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:u24 -s 2 -c 1 -o /tmp/${t}_u24 -f python tools/c3_diag.py mistral 2048 > /dev/null 2>&1; echo "u24 ncu rc $?"
python tools/ncu_summary.py /tmp/${t}_u24.ncu-rep 1024 > $o/${t}_u24_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:probe_exact -c 2 -o /tmp/${t}_probe -f env C1=0 python tools/prefill_bench.py 1 > /dev/null 2>&1; echo "probe ncu rc $?"
ncu -i /tmp/${t}_probe.ncu-rep --page raw --csv > /tmp/${t}_probe_raw.csv 2>&1
python - "$t" <<'PY'
import csv, io, sys
t = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/{t}_probe_raw.csv")))
h = rows[0]
keep = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
with open(f"gpurun_out/{t}_probe_summary.txt", "w") as f:
    for r in rows[2:]:
        for k in keep:
            if k in h:
                f.write(f"{k:70s} {r[h.index(k)][:90]}\n")
        f.write("\n")
PY
du -sh $o
