mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/g12_pytest.log 2>&1; echo pytest rc=$?
tail -16 gpurun_out/g12_pytest.log
timeout 1500 python bench.py > gpurun_out/g12_b8m.log 2>&1; echo b8m rc=$?
tail -c 5000 gpurun_out/g12_b8m.log
timeout 1500 python bench.py --impl reference > gpurun_out/g12_ref.log 2>&1; echo ref rc=$?
tail -c 2500 gpurun_out/g12_ref.log
