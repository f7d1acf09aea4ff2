o=gpurun_out; mkdir -p $o
for cfg in "" "RDKV_DECODE_CTAS=2" "RDKV_DECODE_CTAS=4" "RDKV_DECODE_CTA=1" "RDKV_DECODE_NULL=1" "RDKV_DECODE_NULL=1 RDKV_DECODE_CTAS=2"; do
  env $cfg timeout 300 python tools/u2x_exp.py 200 2>&1 | tail -1
done > $o/r2g_exp.log
cat $o/r2g_exp.log
