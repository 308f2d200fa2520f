set -x; cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v3.json 2> gpurun_out/bench_v3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_frame -s 1 -c 1 -o gpurun_out/prof_frame_v3 python bench.py --steps 1 --warmup 1 --profile > gpurun_out/ncu_v3.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_v3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['msamples_per_s'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
"
