mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g1_pytest.log
timeout 900 python bench.py --n 1000000 --steps 10 --warmup 3 > gpurun_out/g1_b1m.log 2>&1; echo b1m rc=$?
tail -c 3000 gpurun_out/g1_b1m.log
timeout 1500 python bench.py > gpurun_out/g1_b8m.log 2>&1; echo b8m rc=$?
tail -c 4000 gpurun_out/g1_b8m.log
