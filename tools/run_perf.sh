# usage: gpurun -- bash tools/run_perf.sh TAG
#   CFGS="c3 c2" (configs to profile), QUICK=1 (profiles only: no pytest / smoke / bench)
# -> gpurun_out/{pytest_gpu,smoke,bench}_TAG.*, launches_CFG_TAG.csv (ncu launch list of an
#    8-view orbit: warm-up frame, 8 timed frames, 8 byte-counting frames), prof_CFG_TAG.ncu-rep
#    (ncu --set full of the first timed frame's k_warp, k_walk and k_walk2: view 0)
set -x; cd "${GRAFT_REPO_ROOT:-.}"; TAG=${1:-v}
mkdir -p gpurun_out
if [ -z "$QUICK" ]; then
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
fi
for CFG in ${CFGS:-c3 c2}; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_classify|k_walk|k_route|k_short|k_warp|k_iso|Select|Compact" --csv \
  --log-file gpurun_out/launches_${CFG}_$TAG.csv python bench.py --config $CFG --secondary "" --extra "" --steps 8 --warmup 1 --profile > gpurun_out/ncu_launch_${CFG}_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_walk" -s 3 -c 3 \
  -o gpurun_out/prof_${CFG}_$TAG python bench.py --config $CFG --secondary "" --extra "" --steps 8 --warmup 1 --profile > gpurun_out/ncu_${CFG}_$TAG.log 2>&1
done
[ -z "$QUICK" ] && tail -c 600 gpurun_out/bench_$TAG.json
true
