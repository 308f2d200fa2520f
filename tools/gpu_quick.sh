cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_synth.py -q -m gpu -x --timeout 600 > gpurun_out/pt_synth1.log 2>&1; tail -15 gpurun_out/pt_synth1.log
