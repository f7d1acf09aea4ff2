o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_mma.py -x -q > $o/r2h_pytest.log 2>&1; echo "pytest rc $?"; tail -3 $o/r2h_pytest.log
timeout 300 python tools/graph_step.py 200 2>&1 | tail -1
for ppc in 0 1 2; do
  RDKV_DECODE_U24_PPC=$ppc timeout 600 python tools/c3_bench.py --exp qwen2.5-7b_n1024 qwen2.5-7b_n256 mistral-7b_n2048 2>&1 | sed "s/^/ppc$ppc /"
done > $o/r2h_c3.log; cat $o/r2h_c3.log | cut -c1-200
RDKV_DECODE_CTAS=8 timeout 300 python tools/u2x_exp.py 200 2>&1 | tail -1
