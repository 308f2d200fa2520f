# usage: gpurun -- bash tools/prof_libs.sh "c3 c2" VIEW alt/libA.so ...  (the in-tree lib is "cur")
# Per-kernel device times (ncu launch list, serialised) of 3 frames of one view per library.
cd "${GRAFT_REPO_ROOT:-.}"; CFGS=$1; VIEW=$2; shift 2; export XB_CELL_CACHE=/tmp/xb_cells
for c in $CFGS; do for L in cur "$@"; do
echo "== $c view $VIEW $L"
if [ "$L" = cur ]; then unset XB_LIB; else export XB_LIB=$L; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|Select" -c 80 --csv \
  python tools/frames.py $c "" 3 $VIEW 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=collections.defaultdict(list)
for r in rows[1:]:
    t[r[ki].split('(')[0].split('<')[0].replace('void ','')].append(float(r[vi].replace(',','')))
for k,v in t.items():
    if len(v) >= 3: print(f'{k:30s} n={len(v):3d} last3={sum(v[-3:])/3e3:9.1f} us')
"
done; done; unset XB_LIB
