# scan-kernel diagnostics (timing only): ablation switches x ring depth x rank split
set -u
mkdir -p gpurun_out
make -j8 all > gpurun_out/d_build.log 2>&1 || { tail -20 gpurun_out/d_build.log; exit 1; }
CONFIGS=${CONFIGS:-0,256,264,260,272,280} NPROBES=${NPROBES:-32} STAGES=${STAGES:-0,2,3,4,6} SPLITS=${SPLITS:-1,0} \
  timeout 900 python tools/scan_exp.py > gpurun_out/d_abl2.txt 2>&1
tail -3 gpurun_out/d_abl2.txt
