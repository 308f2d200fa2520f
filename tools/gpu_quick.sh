cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match or tiled" > gpurun_out/pt_sh4.log 2>&1; tail -1 gpurun_out/pt_sh4.log
for c in c3 c5 c2; do timeout 300 python tools/ab.py $c warp,noshort 6 > gpurun_out/ab_sh4_$c.log 2>&1; grep median gpurun_out/ab_sh4_$c.log; done
