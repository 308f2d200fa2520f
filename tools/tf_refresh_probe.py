"""Config 4's TF-edit refresh (build_volume_bvh for a new ramp) at a bench config:
python tools/tf_refresh_probe.py c3 [reps] -> per call: Python wall ms, the library's
own build_ms (around build_active), alternating two ramps."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.accel import build_volume_bvh  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
del cells
tfs = [bench.tf_for(model.value_range(0), cfg, max_alpha=a) for a in (0.3, 0.5)]
keep = []
for k in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = build_volume_bvh(regions, tfs[k % 2], 0, model=model)
    t1 = time.perf_counter()
    import ctypes as C

    from paper_2009_03076_b200 import _native as N

    na, ms = C.c_int64(), C.c_double()
    N.check(N.lib().xb_active_info(b.handle.h, C.byref(na), C.byref(ms)))
    print(f"rep {k}: wall {1e3 * (t1 - t0):8.2f} ms  build_active {ms.value:8.2f} ms  active {na.value}", flush=True)
    keep.append(b) if k % 3 == 0 else None  # some results stay alive, others are freed by the next call
