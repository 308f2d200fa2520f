# usage: gpurun -- bash tools/run_perf.sh TAG   (pytest -m gpu, smoke, bench, ncu launch list + full captures)
#   CFGS="c3 c2" (configs to profile), QUICK=1 (profiles only: no pytest / smoke / bench)
set -x; cd "${GRAFT_REPO_ROOT:-.}"; TAG=${1:-v}
mkdir -p gpurun_out
if [ -z "$QUICK" ]; then
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
fi
for CFG in ${CFGS:-c3 c2}; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_classify|k_walk|k_route|k_short|k_warp|k_iso|Select|Compact" -c 60 --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv python bench.py --config $CFG --secondary '' --steps 3 --warmup 1 --profile > gpurun_out/ncu_launch_${CFG}_$TAG.log 2>&1
# -s 4: skip the untimed byte-counting frame (k_walk, k_walk2, k_short, k_warp with COUNT=1)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk|k_short|k_warp" -s 4 -c 4 -o gpurun_out/prof_${CFG}_$TAG python bench.py --config $CFG --secondary '' --steps 1 --warmup 1 --profile > gpurun_out/ncu_${CFG}_$TAG.log 2>&1
done
[ -z "$QUICK" ] && tail -c 600 gpurun_out/bench_$TAG.json
true
