cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2 c3 c5; do XB_PRINT_NCAND=1 timeout 300 python tools/ab.py $c warp 1 2>&1 | grep "candidate" | tail -1; done
