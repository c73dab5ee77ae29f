# ncu capture (source-level) of the k > 32 selection of the GEMM-scan search (GIST-shaped, k = 100)
make -j8 all > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gs_select -s 2 -c 1 -o gpurun_out/gsel python tools/gist_probe.py > gpurun_out/gsel_ncu.log 2>&1; echo "ncu rc=$?"
