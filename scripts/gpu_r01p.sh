#!/bin/bash
O=gpurun_out/r01p
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -c 600 $O/bench.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.jsonl
