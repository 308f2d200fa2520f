# usage: gpurun -- bash tools/sweep_grab.sh : k_warp ray-grab schedule sweep (xb_tuning grab_sm / grab_div / grab_fixed)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
V="warp,k:grab_div=3,k:grab_div=5,k:grab_div=6"
for c in c3 c2 c5 c4; do echo == $c; timeout 900 python tools/ab.py $c "$V" 5 2>&1 | tail -6; done
