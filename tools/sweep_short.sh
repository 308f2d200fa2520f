cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide_short" > gpurun_out/sweep_pytest.log 2>&1; tail -2 gpurun_out/sweep_pytest.log
V="warp,k:short_leaves=12,k:short_leaves=16,k:short_samples=48,k:short_leaves=16+short_samples=48,k:short_leaves=16+short_samples=96,k:short_leaves=4+short_samples=12,k:short_leaves=16+short_samples=48+walk_cap1=24"
for c in c3 c2 c5; do echo == $c; timeout 900 python tools/ab.py $c "$V" 5 2>&1 | tail -8; done
