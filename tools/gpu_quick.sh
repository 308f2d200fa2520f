cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/pt_walk6.log 2>&1; tail -1 gpurun_out/pt_walk6.log
timeout 300 python tools/ab.py c2 warp,nowalk 6 > gpurun_out/ab_walk6.log 2>&1; grep median gpurun_out/ab_walk6.log
timeout 300 python tools/ab.py c3 warp,nowalk 6 > gpurun_out/ab_walk6c3.log 2>&1; grep median gpurun_out/ab_walk6c3.log
