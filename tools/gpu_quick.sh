cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match or tiled or two_cell or opaque or space or iso_hits" > gpurun_out/pt_short.log 2>&1; tail -3 gpurun_out/pt_short.log
for c in c2 c3 c5; do timeout 300 python tools/ab.py $c warp,noshort 6 > gpurun_out/ab_short_$c.log 2>&1; grep median gpurun_out/ab_short_$c.log; done
