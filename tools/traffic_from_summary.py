"""profiles/traffic_<cfg>.json from an ncu summary (tools/ncu_summary.py output):
DRAM bytes (read + write) per launch of the dominant kernel (k_warp) and of the
other captured frame kernels, for one timed frame.
python tools/traffic_from_summary.py profiles/r02_v10_ncu_c3.txt c3"""
import json
import re
import sys

path, cfg = sys.argv[1], sys.argv[2]
per = {}
kern = None
for ln in open(path):
    m = re.match(r"kernel: (.*)", ln)
    if m:
        kern = m.group(1).split("(")[0].replace("void ", "").strip()
        per.setdefault(kern, [])
        per[kern].append(0.0)
        continue
    m = re.match(r"\s+dram__bytes_(read|write)\.sum\s+([\d.]+) (Mbyte|Kbyte|Gbyte|byte)", ln)
    if m and kern:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m.group(3)]
        per[kern][-1] += float(m.group(2)) * scale
# one launch of each kernel (the last capture of each: the timed frame's); the
# bench's roofline.traffic is the dominant kernel's (k_warp), like roofline.achieved
frame = {k: v[-1] for k, v in per.items()}
warp = [k for k in frame if k.startswith("k_warp")]
json.dump({"config": cfg, "kernel": warp[0] if warp else None,
           "dram_bytes_per_launch": int(frame[warp[0]]) if warp else None,
           "per_kernel": {k: int(v) for k, v in frame.items()},
           "frame_dram_bytes": int(sum(frame.values())),
           "source": f"{path} (dram__bytes_read.sum + dram__bytes_write.sum of one launch, ncu --set full "
                     "--clock-control none, orbit view 0 of bench.py --profile)"},
          open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
print(open(f"profiles/traffic_{cfg}.json").read())
