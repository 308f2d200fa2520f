# usage: gpurun -- bash tools/sweep_grab.sh : k_warp ray-grab schedule sweep (xb_tuning grab_sm / grab_div / grab_fixed)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
V="warp,k:grab_sm=0,k:grab_div=2,k:grab_div=8,k:grab_div=1,k:grab_fixed=2"
for c in c3 c2 c5 c4; do echo == $c; timeout 900 python tools/ab.py $c "$V" 5 2>&1 | tail -6; done
