make -j8 all > gpurun_out/q5_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q5_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q5_pytest.log
timeout 600 python tools/param_grids.py --search-only --out gpurun_out/q5_grids.json 2>&1 | tail -20
