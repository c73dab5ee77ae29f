mkdir -p gpurun_out
CONFIGS=0,1 NPROBES=32 SPLITS=0,1,2,3,4,6,12,16 timeout 300 python tools/scan_exp.py > gpurun_out/r02n_scanexp.txt 2>&1
cat gpurun_out/r02n_scanexp.txt
