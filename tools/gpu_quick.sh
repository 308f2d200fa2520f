cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
for c in c3 c2 c5 c4; do echo $c; python tools/ab.py $c "warp" 2>&1 | tail -1 | cut -c1-70; XB_LIB=alt/libexabricks_head.so python tools/ab.py $c "warp" 2>&1 | tail -1 | cut -c1-70; done
