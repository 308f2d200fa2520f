cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c2; do
for v in "k:fuse_short=1" "k:fuse_short=0+short_rays=1"; do
echo "== $c $v"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_classify|k_walk|k_route|k_short|k_warp|k_iso|Select" -c 60 --csv python tools/frames.py $c "$v" 3 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=collections.defaultdict(list)
for r in rows[1:]:
    t[r[ki].split('(')[0].split('<')[0]].append(float(r[vi].replace(',','')))
for k,v in t.items(): print(f'{k:30s} n={len(v):3d} last={v[-1]/1e3:9.1f} us')
"
done; done
