o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > $o/r2i_pytest.log 2>&1; echo "pytest rc $?"; tail -3 $o/r2i_pytest.log
timeout 600 python tools/prefill_bench.py 3 > $o/r2i_prefill.log 2>&1; echo "prefill rc $?"; tail -3 $o/r2i_prefill.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $o/r2i_prefill_ncu.csv env C1=0 python tools/prefill_bench.py 1 > $o/r2i_prefill_ncu.log 2>&1; echo "prefill ncu rc $?"
