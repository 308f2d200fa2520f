cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "acceptance or frames_match or tiled or iso" 2>&1 | tail -3
python tools/ab.py c4 warp,frame 2>&1 | tail -4
XB_ISO_LANE=1 python tools/ab.py c4 warp 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_iso|k_classify|k_walk|k_short|k_warp" -c 40 --csv --log-file gpurun_out/launch_c4b.csv python bench.py --config c4 --secondary '' --steps 2 --warmup 1 --profile > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launch_c4b.csv')))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
ki,vi=h.index("Kernel Name"),h.index("Metric Value")
t=[]
for r in rows[hi+1:]:
    try: t.append((r[ki][:40], round(float(r[vi])/1e3)))
    except: pass
for x in t[-12:]: print(x)
PY
