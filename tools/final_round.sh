# final evidence of the round: GPU suite, bench line, step launch list, scan ncu capture, §4.3 grid
set -u
TAG=${1:-r03c}
mkdir -p gpurun_out
bash tools/gpu_round.sh $TAG tests bench launches full
timeout 600 python tools/param_grids.py --search-only --quick --out gpurun_out/${TAG}_grids_search.json > gpurun_out/${TAG}_grids.log 2>&1
echo "grids rc=$?"; tail -6 gpurun_out/${TAG}_grids.log
