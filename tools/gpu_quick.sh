cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "frames_match or acceptance or two_cell or space_skipping or iso_hits or opaque" > gpurun_out/pt_warp10.log 2>&1; tail -3 gpurun_out/pt_warp10.log
timeout 300 python tools/ab.py c2 warp,frame 10 > gpurun_out/ab14.log 2>&1; tail -4 gpurun_out/ab14.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 1 -c 1 -o gpurun_out/prof_warp14 python bench.py --steps 1 --warmup 1 --profile > gpurun_out/ncu_warp14.log 2>&1; tail -1 gpurun_out/ncu_warp14.log
