mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/g2_pytest.log
timeout 1200 python scripts/kernel_table.py --n 8000000 > gpurun_out/g2_kt_ls.log 2>&1; echo kt rc=$?
tail -c 2500 gpurun_out/g2_kt_ls.log
RSB_TRSV_GRID=syncfree timeout 600 python scripts/kernel_table.py --n 8000000 > gpurun_out/g2_kt_sf.log 2>&1; echo kt2 rc=$?
tail -c 2500 gpurun_out/g2_kt_sf.log
timeout 900 python bench.py --no-tol > gpurun_out/g2_b8m.log 2>&1; echo b8m rc=$?
tail -c 3000 gpurun_out/g2_b8m.log
