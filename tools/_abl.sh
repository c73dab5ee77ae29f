mkdir -p gpurun_out
for i in 1 2; do
SIVF_LIB_PATH=build/libsivf_old.so CONFIGS=0 NPROBES=32 timeout 300 python tools/scan_exp.py 2>&1 | grep nprobe | sed 's/^/old /'
CONFIGS=0 NPROBES=32 timeout 300 python tools/scan_exp.py 2>&1 | grep nprobe | sed 's/^/tpl /'
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02zm_pytest.txt 2>&1; tail -2 gpurun_out/r02zm_pytest.txt
