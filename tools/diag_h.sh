make -j8 all build/libsivf_proft.so > /dev/null 2>&1 || exit 1
SIVF_LIB_PATH=build/libsivf_proft.so G=8 NITER=4 timeout 600 python tools/trace_h.py 2>&1 | grep "blk 0 warp" | sort -t' ' -k4 -n | tail -16
