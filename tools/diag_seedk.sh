make -j8 all > /dev/null 2>&1 || exit 1
CONFIGS=0 NPROBES=32 STAGES=0 SPLITS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_seed_list -s 3 -c 1 -o gpurun_out/seedk python tools/scan_exp.py > gpurun_out/seedk.log 2>&1; echo "ncu rc=$?"
