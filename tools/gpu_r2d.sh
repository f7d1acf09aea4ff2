o=gpurun_out; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "configs3" > $o/r2d_pytest.log 2>&1; echo "pytest rc $?"; tail -15 $o/r2d_pytest.log
timeout 900 python tools/c3_bench.py > $o/r2d_c3.log 2>&1; echo "c3 rc $?"; cat $o/r2d_c3.log | tail -8
