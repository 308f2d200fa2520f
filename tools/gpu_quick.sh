cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
for c in c3 c2 c4 c5; do echo $c; python tools/ab.py $c warp,frame 10 2>&1 | tail -2 | cut -c1-60; done
