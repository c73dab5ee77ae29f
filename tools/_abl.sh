mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02zc_pytest.txt 2>&1; tail -2 gpurun_out/r02zc_pytest.txt
timeout 600 python tools/gist_probe.py 2>&1 | grep gist
