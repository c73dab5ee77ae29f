mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02w_pytest.txt 2>&1; tail -2 gpurun_out/r02w_pytest.txt
HIST=1 SIVF_LIB_PATH=build/libsivf_prof.so timeout 300 python tools/coarse_probe.py 2>&1 | grep -v "^blk" | tail -3
timeout 300 python tools/coarse_probe.py 2>&1 | grep SEL
NPROBE=8 timeout 300 python tools/coarse_probe.py 2>&1 | grep SEL
