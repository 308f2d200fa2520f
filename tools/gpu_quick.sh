cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match or tiled or two_cell or opaque or space or iso_hits" > gpurun_out/pt_eng.log 2>&1; tail -3 gpurun_out/pt_eng.log
timeout 300 python tools/ab.py c2 warp,nowalk 6 > gpurun_out/ab_eng.log 2>&1; grep median gpurun_out/ab_eng.log
timeout 300 python tools/ab.py c3 warp 6 > gpurun_out/ab_eng3.log 2>&1; grep median gpurun_out/ab_eng3.log
