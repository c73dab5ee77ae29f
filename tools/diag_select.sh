# coarse selection diagnostics: per-phase clocks (prof build) + ncu full capture of k_coarse_select<32,1>
set -u
mkdir -p gpurun_out
make -j8 all build/libsivf_prof.so > /dev/null 2>&1 || exit 1
HIST=1 SIVF_LIB_PATH=build/libsivf_prof.so timeout 300 python tools/coarse_probe.py 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_coarse_select" -s 2 -c 2 \
  -o gpurun_out/sel python tools/coarse_probe.py > gpurun_out/sel_ncu.log 2>&1; echo "ncu rc=$?"
