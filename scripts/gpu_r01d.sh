#!/bin/bash
O=gpurun_out/r01d
mkdir -p $O
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_configs.py -x -q -k "config3" > $O/sanitize_default.log 2>&1; echo rc=$? >> $O/sanitize_default.log
RSB_TRSV_GRID=lsync timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_configs.py -x -q -k "config3" > $O/sanitize_lsync.log 2>&1; echo rc=$? >> $O/sanitize_lsync.log
tail -3 $O/sanitize_*.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
RSB_TRSV_GRID=lsync timeout 900 python scripts/microbench_trsv.py --config 4 --n 2000000 > $O/trsv_lsync_2m.json 2>&1
cat $O/trsv_*.json
