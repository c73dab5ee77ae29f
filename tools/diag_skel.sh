# scan control-skeleton ablation (timing only): which role sets the 0.17 ms floor
make -j8 all > /dev/null 2>&1 || exit 1
# 256 idle epilogue, 4 no MMA, 8 no B copies, 16 no A loads, 512 meta forwards only
CONFIGS=${CONFIGS:-256,260,268,284,796,780,772,764} NPROBES=32 STAGES=0 SPLITS=1 timeout 600 python tools/scan_exp.py 2>&1 | cut -c1-70
