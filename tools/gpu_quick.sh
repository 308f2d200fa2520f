cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c2; do timeout 300 python tools/ab.py $c warp,sl4_16,sl8_16,sl8_48,sl16_32,sl16_64,sl32_64 6 > gpurun_out/ab_sl_$c.log 2>&1; grep median gpurun_out/ab_sl_$c.log; done
