cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match" > gpurun_out/pt_res1.log 2>&1; tail -1 gpurun_out/pt_res1.log
timeout 300 python tools/ab.py c2 warp,cap16,cap32,cap128,nowalk 6 > gpurun_out/ab_res1.log 2>&1; grep median gpurun_out/ab_res1.log
timeout 300 python tools/ab.py c3 warp,cap16,cap32,cap128,nowalk 6 > gpurun_out/ab_res1c3.log 2>&1; grep median gpurun_out/ab_res1c3.log
