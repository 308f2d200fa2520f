"""Oracle digests of the builders at the benchmarked scales (test fixture).

  python tools/make_scale_digests.py c2 c3
  XB_DIGESTS_OUT=gpurun_out/scale_digests_c5.json python tools/make_scale_digests.py c5   # on the GPU box (RAM)

For each bench config: the cells from the numpy generator (bit-exact
restatement of the reference's generate_synthetic, R/io.py:247-295, pinned by
tests/golden/digests.json), then the C oracle's build_bricks / build_regions
(oracle/xb_oracle.c, pinned to the reference's golden arrays).  sha256 of every
array (tests/tests_util.py:sha) -> tests/golden/scale_digests.json, which
bench.py and tests/test_gpu_scale.py compare the GPU builders against."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import oracle  # noqa: E402
from tests_util import sha  # noqa: E402

OUT = Path(os.environ.get("XB_DIGESTS_OUT", ROOT / "tests" / "golden" / "scale_digests.json"))
MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")


def main():
    db = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in sys.argv[1:]:
        cfg = bench.CONFIGS[name]
        t0 = time.time()
        cells = bench.make_cells(dict(cfg, gpu_gen=False), host=True)  # the numpy generator
        t1 = time.time()
        m = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
        t2 = time.time()
        r = oracle.build_regions(*(m[k] for k in MODEL_KEYS))
        t3 = time.time()
        d = {"n_cells": len(cells), "n_bricks": int(len(m["brick_level"])), "n_regions": int(len(r["finest_width"])),
             "cells": {a: sha(getattr(cells, a)) for a in ("i", "j", "k", "level", "values")},
             "model": {k: sha(m[k]) for k in MODEL_KEYS}, "regions": {k: sha(r[k]) for k in REGION_KEYS},
             "seconds": {"generate": round(t1 - t0, 1), "oracle_bricks": round(t2 - t1, 1),
                         "oracle_regions": round(t3 - t2, 1)}}
        db[name] = d
        print(name, json.dumps(d["seconds"]), d["n_cells"], d["n_bricks"], d["n_regions"], flush=True)
        OUT.write_text(json.dumps(db, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
