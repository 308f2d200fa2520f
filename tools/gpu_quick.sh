cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/ab.py c2 warp,warp3,warp5,f4,f16,cap96 6 > gpurun_out/ab_t1.log 2>&1; grep median gpurun_out/ab_t1.log
timeout 300 python tools/ab.py c3 warp,warp3,warp5,f4,f16,cap96 6 > gpurun_out/ab_t1c3.log 2>&1; grep median gpurun_out/ab_t1c3.log
