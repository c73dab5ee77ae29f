mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/concurrency_stress.py 1 8 2000 > gpurun_out/r02zk_racecheck.txt 2>&1; tail -4 gpurun_out/r02zk_racecheck.txt
timeout 1200 compute-sanitizer --tool synccheck python tools/concurrency_stress.py 1 8 2000 > gpurun_out/r02zk_synccheck.txt 2>&1; tail -3 gpurun_out/r02zk_synccheck.txt
