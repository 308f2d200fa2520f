cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "lbvh or traversal or acceptance or frames_match" > gpurun_out/pt_lbvh1.log 2>&1; tail -25 gpurun_out/pt_lbvh1.log
