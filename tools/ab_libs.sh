# usage: gpurun -- bash tools/ab_libs.sh "c3 c2" alt/libA.so alt/libB.so ...  (the in-tree lib is timed as "cur")
# Interleaves whole-process runs of tools/ab.py per library and config.
cd "${GRAFT_REPO_ROOT:-.}"; CFGS=$1; shift; export XB_CELL_CACHE=/tmp/xb_cells
for rep in 1 2; do for c in $CFGS; do
  echo "== $c cur"; timeout 600 python tools/ab.py $c warp 15 2>&1 | tail -1 | cut -c1-100
  for L in "$@"; do echo "== $c $L"; XB_LIB=$L timeout 600 python tools/ab.py $c warp 15 2>&1 | tail -1 | cut -c1-100; done
done; done
