#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list, ncu full capture of the scan.
# usage (under gpurun): bash tools/gpu_round.sh [tag] [what...]   what in {tests,bench,launches,full}
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-tests bench launches full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
make -j8 all > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1
      echo "pytest gpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log ;;
    bench)
      timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
      echo "bench rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra \
        > gpurun_out/${TAG}_launches_bench.json 2> gpurun_out/${TAG}_launches.err
      echo "launches rc=$?" ;;
    full)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 1 -c 1 \
        -o gpurun_out/${TAG}_scan python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-extra \
        > gpurun_out/${TAG}_full_bench.json 2> gpurun_out/${TAG}_full.err
      echo "full rc=$?" ;;
  esac
done
