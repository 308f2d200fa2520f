cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --secondary '' --no-cpu-baseline > gpurun_out/bench_pin.json 2> gpurun_out/bench_pin.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_pin.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "frames_match" > gpurun_out/pt_pin.log 2>&1; tail -1 gpurun_out/pt_pin.log
