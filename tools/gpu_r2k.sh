o=gpurun_out; mkdir -p $o
timeout 120 tools/tc05/tc05_core 4096 > $o/r2k_tc05.log 2>&1; echo "tc05 rc $?"; cat $o/r2k_tc05.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --csv --log-file $o/r2k_tc05_ncu.csv tools/tc05/tc05_core 1024 > /dev/null 2>&1; echo "ncu rc $?"
timeout 600 python -m pytest tests/test_gpu_dropin.py -q > $o/r2k_dropin.log 2>&1; echo "dropin rc $?"; tail -3 $o/r2k_dropin.log
