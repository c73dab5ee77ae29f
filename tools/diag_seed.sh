# seed / rank-split sweeps of the scan (timing only)
make -j8 all > /dev/null 2>&1
CONFIGS=0 SEEDS=${SEEDS:-0} NPROBES=${NPROBES:-32,8} STAGES=0 SPLITS=${SPLITS:-1,2,4,6} timeout 600 python tools/scan_exp.py 2>&1 | cut -c1-100
