o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_mma.py -x -q > $o/r2f_pytest.log 2>&1; echo "pytest rc $?"; tail -4 $o/r2f_pytest.log
timeout 900 python tools/c3_bench.py > $o/r2f_c3.log 2>&1; echo "c3 rc $?"; cat $o/r2f_c3.log | tail -8
timeout 600 ncu --set full --import-source on --clock-control none -k regex:u24 -s 2 -c 1 -o $o/r2f_u24_q1024 -f python tools/c3_diag.py qwen 1024 > $o/r2f_ncu.log 2>&1; echo "ncu rc $?"
