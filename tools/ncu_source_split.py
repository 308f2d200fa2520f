"""Split a kernel's ncu warp-stall samples and executed instructions by source
ranges: ncu -i REP --kernel-name regex:k_warp --page source --csv
--print-source cuda,sass > src.csv; python tools/ncu_source_split.py src.csv
'{"name": ["render.cu", first_line, last_line], ...}' (line numbers of the
source embedded in the report)."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; fpath = None; data = collections.defaultdict(float); inst = collections.defaultdict(float)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fpath = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == "Function Name": continue
    if r and r[0] == "Line No": hdr = r; si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed"); continue
    if hdr and r and r[0].strip().isdigit():
        try: v = float(r[si] or 0); w = float(r[ii] or 0)
        except ValueError: continue
        data[(fpath, int(r[0]))] += v; inst[(fpath, int(r[0]))] += w
tot = sum(data.values()); ti = sum(inst.values())
print("total samples", tot, "instructions", ti)
def rng(f, a, b): return sum(v for (ff, l), v in data.items() if ff == f and a <= l <= b), sum(v for (ff, l), v in inst.items() if ff == f and a <= l <= b)
import json
cats = json.loads(sys.argv[2])
acc = 0
for name, (f, a, b) in cats.items():
    s, i = rng(f, a, b); acc += s
    print(f"{name:28s} stall-samples {100*s/tot:5.1f} %  instr {100*i/ti:5.1f} %")
print("other", 100*(tot-acc)/tot)
top = sorted(data.items(), key=lambda kv: -kv[1])[:25]
for (f, l), v in top: print(f"{f}:{l} {100*v/tot:5.2f} %")
