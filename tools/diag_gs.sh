# ncu capture of the GEMM scan (GIST-shaped k=100 search)
make -j8 all > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none -k regex:k_scan_gs -s 2 -c 1 -o gpurun_out/gs python tools/gist_probe.py > gpurun_out/gs_ncu.log 2>&1; echo "ncu rc=$?"
