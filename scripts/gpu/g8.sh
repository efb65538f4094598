mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/g8_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g8_pytest.log
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_launches.csv python scripts/batch_profile.py --n 8000000 --iters 2 > gpurun_out/g8.log 2>&1; echo ncu rc=$?
timeout 1200 python bench.py --no-tol --no-parity > gpurun_out/g8_b8m.log 2>&1; echo b8m rc=$?
tail -c 1500 gpurun_out/g8_b8m.log
