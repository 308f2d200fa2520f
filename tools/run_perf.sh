# usage: gpurun -- bash tools/run_perf.sh TAG   (pytest -m gpu, bench, ncu launch list + full capture of k_frame)
set -x; cd "${GRAFT_REPO_ROOT:-.}"; TAG=${1:-v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_frame -s 1 -c 1 -o gpurun_out/prof_frame_$TAG python bench.py --steps 1 --warmup 1 --profile > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.json
