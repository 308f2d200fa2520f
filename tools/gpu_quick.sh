cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c2 c5 c4; do echo $c; python tools/ab.py $c "warp,short,noshort,sl12_32,sl16_48" 2>&1 | tail -5 | cut -c1-70; done
