#!/bin/bash
# full validation pass (round 2): tests, smoke, bench, 2-rank torchrun, ncu evidence
o=gpurun_out; mkdir -p $o; t=r2l
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/${t}_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $o/${t}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 $o/${t}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${t}_smoke.log 2>&1; echo "smoke rc $?"
timeout 1500 python bench.py > $o/${t}_bench.json 2> $o/${t}_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > $o/${t}_bench_ref.json 2> $o/${t}_bench_ref.err; echo "ref rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --dist-backend gloo --no-secondary --no-fp16-baseline --no-pipeline > $o/${t}_torchrun2.json 2> $o/${t}_torchrun2.err; echo "torchrun rc $?"
timeout 600 python tools/graph_step.py 200 > $o/${t}_graph_plain.log 2>&1
timeout 900 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $o/${t}_graph_ncu.csv python tools/graph_step.py 200 > /dev/null 2>&1; echo "graph ncu rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_u2x -s 3 -c 1 -o $o/${t}_u2x -f python tools/graph_step.py 10 > /dev/null 2>&1; echo "u2x ncu rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:u24 -s 2 -c 1 -o $o/${t}_u24 -f python tools/c3_diag.py mistral 2048 > /dev/null 2>&1; echo "u24 ncu rc $?"
timeout 600 ncu --set full --clock-control none -k regex:probe_exact -c 2 -o $o/${t}_probe -f env C1=0 python tools/prefill_bench.py 1 > /dev/null 2>&1; echo "probe ncu rc $?"
timeout 900 python tools/c3_bench.py > $o/${t}_c3.log 2>&1; echo "c3 rc $?"
