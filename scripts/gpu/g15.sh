mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k "row_partitioned" > gpurun_out/g15_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/g15_pytest.log
timeout 1500 python bench.py --partition rows --steps 10 --warmup 2 > gpurun_out/g15_rows.log 2>&1; echo rows rc=$?
tail -c 1500 gpurun_out/g15_rows.log
