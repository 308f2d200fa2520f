cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c2 c5; do timeout 300 python tools/ab.py $c warp,w2_16_64,w2_16_96,w2_16_128,w2_24_64 6 > gpurun_out/ab_w3_$c.log 2>&1; grep median gpurun_out/ab_w3_$c.log; done
