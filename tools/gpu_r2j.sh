o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_dropin.py -q > $o/r2j_pytest.log 2>&1; echo "pytest rc $?"; tail -5 $o/r2j_pytest.log
timeout 600 python tools/prefill_bench.py 3 > $o/r2j_prefill.log 2>&1; echo "prefill rc $?"; tail -3 $o/r2j_prefill.log
