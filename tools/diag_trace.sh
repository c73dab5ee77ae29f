# k_scan_tc block-0 traces under ablation switches (prof timing build)
set -u
mkdir -p gpurun_out
make -j8 all build/libsivf_proft.so > gpurun_out/t_build.log 2>&1 || { tail -20 gpurun_out/t_build.log; exit 1; }
for d in ${DBGS:-256 260 0}; do
  SIVF_LIB_PATH=build/libsivf_proft.so DBG=$d timeout 300 python tools/trace_scan.py > gpurun_out/t_trace_$d.txt 2>&1
done
