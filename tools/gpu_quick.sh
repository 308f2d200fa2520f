cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c2 c5; do echo $c; python tools/ab.py $c "warp,e:XB_FUSE_SHORT=0" 2>&1 | tail -2 | cut -c1-70; XB_LIB=alt/libexabricks_head.so python tools/ab.py $c "warp" 2>&1 | tail -1 | cut -c1-70; python tools/ab.py $c "warp" 2>&1 | tail -1 | cut -c1-70; done
