mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02zh_pytest.txt 2>&1; tail -2 gpurun_out/r02zh_pytest.txt
