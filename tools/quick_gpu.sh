# build + GPU suite + scan ablation (timing) in one call
set -u
mkdir -p gpurun_out
T=${TAG:-q}
make -j8 all > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
CONFIGS=${CONFIGS:-0,1,256,260} NPROBES=${NPROBES:-32,8} STAGES=0 SPLITS=${SPLITS:-1} timeout 600 python tools/scan_exp.py > gpurun_out/${T}_abl.txt 2>&1
cat gpurun_out/${T}_abl.txt | cut -c1-90
