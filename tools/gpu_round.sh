#!/bin/bash
# tools: one GPU-box pass — gpu tests, smoke, bench, graph-level ncu timing and a
# full ncu capture of the headline decode kernel. Usage: tools/gpu_round.sh TAG [parts]
# parts: any of t (tests) s (smoke) b (bench) g (graph ncu) f (full ncu) l (launch list)
tag=${1:-r2}; parts=${2:-tsbgfl}
o=gpurun_out
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/${tag}_gpu.txt 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' >> $o/${tag}_gpu.txt
if [[ $parts == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $o/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> $o/${tag}_pytest.log
  tail -3 $o/${tag}_pytest.log
fi
if [[ $parts == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc $?"
fi
if [[ $parts == *b* ]]; then
  timeout 1200 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench rc $?"
  tail -c 600 $o/${tag}_bench.json
fi
if [[ $parts == *g* ]]; then
  timeout 600 python tools/graph_step.py 200 > $o/${tag}_graph_plain.log 2>&1
  timeout 900 ncu --graph-profiling graph --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $o/${tag}_graph_ncu.csv python tools/graph_step.py 200 > $o/${tag}_graph_ncu.log 2>&1
  echo "graph ncu rc $?"; cat $o/${tag}_graph_plain.log | tail -2
fi
if [[ $parts == *l* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $o/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-fp16-baseline \
    --no-cpu-baseline > $o/${tag}_launches.log 2>&1; echo "launch list rc $?"
fi
if [[ $parts == *f* ]]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_u2x -s 3 -c 1 \
    -o $o/${tag}_u2x -f python tools/graph_step.py 10 > $o/${tag}_u2x.log 2>&1; echo "full ncu rc $?"
fi
