o=gpurun_out; mkdir -p $o
timeout 300 python tools/c3_diag.py qwen 1024 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:u24 -s 2 -c 1 -o $o/r2e_u24_q256 -f python tools/c3_diag.py qwen 256 > $o/r2e_ncu.log 2>&1; echo "ncu rc $?"; tail -2 $o/r2e_ncu.log
