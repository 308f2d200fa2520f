"""Builder timing spread at a bench config: python tools/build_probe.py c3 [reps]
-> per rep: build_bricks and build_regions wall ms (host cells uploaded each time)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cells = bench.make_cells(cfg)
for k in range(reps):
    torch.cuda.synchronize()
    ta = time.perf_counter()
    model, _ = build_bricks(cells)
    tb = time.perf_counter()
    regions = build_regions(model)
    tc = time.perf_counter()
    print(f"rep {k}: bricks {1e3 * (tb - ta):8.1f} ms  regions {1e3 * (tc - tb):8.1f} ms", flush=True)
    del regions, model
