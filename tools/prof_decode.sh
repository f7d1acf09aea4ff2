#!/bin/bash
# tools: ncu --set full of the decode kernel on the bench workload (run on the GPU box)
# usage: tools/prof_decode.sh NAME [kernel-regex]
name=${1:-u2x}; rx=${2:-decode_u2x}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -c 1 -o gpurun_out/$name -f python tools/decode_sweep.py 0:0 > gpurun_out/$name.log 2>&1
tail -3 gpurun_out/$name.log
