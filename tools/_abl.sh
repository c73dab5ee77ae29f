mkdir -p gpurun_out
CONFIGS=815,831,1,0 NPROBES=32 timeout 300 python tools/scan_exp.py > gpurun_out/r02s_scanexp.txt 2>&1
SIVF_LIB_PATH=build/libsivf_sleep.so CONFIGS=815,831,1,0 NPROBES=32 timeout 300 python tools/scan_exp.py >> gpurun_out/r02s_scanexp.txt 2>&1
cat gpurun_out/r02s_scanexp.txt
