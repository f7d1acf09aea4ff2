o=gpurun_out; mkdir -p $o
timeout 600 python tools/zc_sweep.py > $o/r2p_zc_default.log 2>&1; tail -1 $o/r2p_zc_default.log
RDKV_DECODE_PAIRS=6 timeout 600 python tools/zc_sweep.py --exp > $o/r2p_zc_p6.log 2>&1; tail -1 $o/r2p_zc_p6.log
RDKV_DECODE_PAIRS=4 timeout 600 python tools/zc_sweep.py --exp > $o/r2p_zc_p4.log 2>&1; tail -1 $o/r2p_zc_p4.log
timeout 600 python -m pytest tests/test_gpu_mma.py -q -k "zone_c or append" > $o/r2p_pytest.log 2>&1; tail -1 $o/r2p_pytest.log
