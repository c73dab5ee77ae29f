# A/B of the scan plan (k_scan_plan): baseline library (build/libsivf_base.so) vs the tree
make -j8 all > /dev/null 2>&1 || exit 1
for lib in build/libsivf_base.so paper_2601_11808_b200/lib/libsivf.so; do
  echo "== $lib"
  SIVF_LIB_PATH=$lib CONFIGS=0 NPROBES=32,8 STAGES=0 SPLITS=1 timeout 300 python tools/scan_exp.py 2>&1 | cut -c1-90
  SIVF_LIB_PATH=$lib G=8 timeout 300 python tools/h_shard_probe.py 2>&1 | tail -1
done
