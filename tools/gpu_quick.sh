cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c5 c4; do timeout 1200 python bench.py --config $c --secondary '' --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); c=d['config']
print('$c', d['value'], d['ms_per_step'], d['msamples_per_s'], c['cells'], c['bricks'], c['regions'], c['build_ms'], c.get('tf_refresh_ms'), d['frame']['samples'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'))"; tail -2 gpurun_out/bench_$c.err; done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
