# GPU suite + per-list seed on/off A/B of the scan (timing only)
make -j8 all > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q11_pytest.log
for sl in 1 0; do SEEDLIST=$sl CONFIGS=0,1 NPROBES=32,16,8 STAGES=0 SPLITS=1 timeout 300 python tools/scan_exp.py 2>&1 | cut -c1-70 | sed "s/^/seedlist=$sl /"; done
