cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match or tiled" > gpurun_out/pt_w4.log 2>&1; tail -3 gpurun_out/pt_w4.log
