#!/bin/bash
# validation pass A (small outputs only): tests, smoke, bench (+ reference arm), 2-rank torchrun, graph-level ncu timing, configs[3]
o=gpurun_out; mkdir -p $o; t=${1:-r2m}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/${t}_gpu.txt 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' >> $o/${t}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $o/${t}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 $o/${t}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${t}_smoke.log 2>&1; echo "smoke rc $?"
timeout 1500 python bench.py > $o/${t}_bench.json 2> $o/${t}_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > $o/${t}_bench_ref.json 2> $o/${t}_bench_ref.err; echo "ref rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --dist-backend gloo --no-secondary --no-fp16-baseline --no-pipeline > $o/${t}_torchrun2.json 2> $o/${t}_torchrun2.err; echo "torchrun rc $?"
timeout 600 python tools/graph_step.py 200 > $o/${t}_graph_plain.log 2>&1
timeout 900 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file /tmp/${t}_graph_ncu.csv python tools/graph_step.py 200 > /dev/null 2>&1; echo "graph ncu rc $?"
grep '"graph"' /tmp/${t}_graph_ncu.csv > $o/${t}_graph_ncu.csv
timeout 900 python tools/c3_bench.py > $o/${t}_c3.log 2>&1; echo "c3 rc $?"
du -sh $o
