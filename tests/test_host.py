"""CPU-side tests: the C ABI library loads and exports every declared symbol,
host logic of the drop-in API matches the reference's known answers, the
synthetic generator reproduces the reference's cells bit-for-bit, file formats
round-trip, and the multi-GPU tile partition is exact."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_digests
from tests_util import sha, spec_from_digest

DIG = golden_digests()["models"]


# ------------------------------------------------------------------ C ABI


def declared_symbols():
    text = (ROOT / "include" / "exabricks.h").read_text()
    return sorted(set(re.findall(r"\b(xb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2009_03076_b200 import _native as N

    lib = N.load_library()
    declared = declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.SIGNATURES), "ctypes signatures out of sync with include/exabricks.h"
    assert lib.xb_abi_version() == 1


def test_struct_layouts_match_header():
    from paper_2009_03076_b200 import _native as N

    # xb_camera: 2 ints + 12 doubles + 2 doubles; xb_march per the header
    assert ctypes.sizeof(N.XbCamera) == 8 + 14 * 8
    assert ctypes.sizeof(N.XbMarch) == 3 * 8 + 8 + 8 + 24 * 8 + 8 + 8 + 3 * 8 + 16 + 1024 * 8 + 8  # + use_tree (padded)


def test_struct_sizes_match_c_compiler(tmp_path):
    """ctypes mirrors of xb_camera / xb_march / xb_synth_spec match gcc's layout of include/exabricks.h."""
    import subprocess

    from paper_2009_03076_b200 import _native as N

    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "exabricks.h"\nint main(void){printf("%zu %zu %zu %zu\\n",'
                   'sizeof(xb_camera), sizeof(xb_march), sizeof(xb_synth_spec), sizeof(xb_tuning));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [ctypes.sizeof(N.XbCamera), ctypes.sizeof(N.XbMarch), ctypes.sizeof(N.XbSynthSpec),
                   ctypes.sizeof(N.XbTuning)]


def test_compute_fails_loudly_without_device():
    """No CPU fallback: without a usable CUDA device the compute API raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.model import CellList

    with pytest.raises(N.NativeUnavailable):
        build_bricks(CellList([0], [0], [0], [0], [1.0]))


# ------------------------------------------------------------------ host helpers vs golden


def test_pixel_rho_and_max_opacity_match_reference():
    from paper_2009_03076_b200.accel import TransferFunction, max_opacity
    from paper_2009_03076_b200.render import pixel_rho

    g = dict(np.load(GOLDEN / "tf_rho.npz"))
    for si, s in enumerate(g["rho_seeds"]):
        got = [pixel_rho(int(p), int(s)) for p in g["rho_pixels"]]
        assert np.array_equal(got, g["rho_values"][si])
    for t in range(len(g["tf_rgba"])):
        tf = TransferFunction(g[f"tf{t}_domain"], g["tf_rgba"][t])
        got = [max_opacity(tf, r) for r in g["tf_ranges"][t]]
        assert np.array_equal(got, g["tf_max_opacity"][t])
    tf = TransferFunction(g["tf0_domain"], g["tf_rgba"][0])
    got = np.array([tf.sample(v) for v in g["tf_sample_values"]])
    assert np.array_equal(got, g["tf_sample_out"])


def test_transfer_function_validation_and_dict():
    from paper_2009_03076_b200.accel import RAMP_SIZE, TransferFunction

    with pytest.raises(ValueError):
        TransferFunction((1.0, 1.0), np.zeros((RAMP_SIZE, 4)))
    with pytest.raises(ValueError):
        TransferFunction((0.0, 1.0), np.zeros((100, 4)))
    with pytest.raises(ValueError):
        TransferFunction((0.0, 1.0), np.full((RAMP_SIZE, 4), 1.5))
    tf = TransferFunction.grayscale((2.0, 4.0), max_alpha=0.5)
    assert np.allclose(tf.sample(3.0), [0.5, 0.5, 0.5, 0.25])
    back = TransferFunction.from_dict(tf.to_dict())
    assert back.domain == tf.domain and np.array_equal(back.rgba, tf.rgba)


def test_intervals_opacity_shade_known_answers():
    from paper_2009_03076_b200.render import make_intervals, opacity_correct, shade

    got = make_intervals(1.0, 2.0, 0.4, 0.0)
    for a, b in zip(got, [(1.0, 1.2), (1.2, 1.6), (1.6, 2.0)]):
        assert a == pytest.approx(b, abs=1e-12)
    assert make_intervals(3.0, 3.1, 5.0, 0.0) == [(3.0, 3.1)]
    assert opacity_correct(0.5, 1.0, 1.0) == 0.5
    assert opacity_correct(0.5, 2.0, 1.0) == 0.75
    c = np.array([1.0, 0.5, 0.25])
    assert np.allclose(shade(c, [0, 0, 2], [0, 0, 1]), c)
    assert np.allclose(shade(c, [0, 0, 0], [0, 0, 1]), 0.2 * c)


def test_camera_and_params_validation():
    from paper_2009_03076_b200.render import Camera, MarchParams

    with pytest.raises(ValueError):
        Camera([0, 0, 0], [0, 1, 0], [0, 1, 0])
    with pytest.raises(ValueError):
        Camera([0, 0, 0], [0, 0, 1], [0, 1, 0], fov_y=180.0)
    for bad in (dict(samples_per_cell=0.0), dict(early_term_threshold=0.0), dict(gradient_mode="sobel"),
                dict(clip_planes=[([1, 0, 0], 0.0)] * 7)):
        with pytest.raises(ValueError):
            MarchParams(**bad)
    cam = Camera([0, 0, 0], [0, 0, 1], [0, 1, 0], 40.0, 101, 101)
    o, d = cam.ray(50, 50)
    assert np.allclose(d, [0, 0, 1], atol=1e-9)


# ------------------------------------------------------------------ data model / formats


@pytest.mark.parametrize("name", sorted(n for n, d in DIG.items() if "spec" in d))
def test_synthetic_generator_reproduces_reference_cells(name):
    from paper_2009_03076_b200 import io as xio

    cl = xio.generate_synthetic(spec_from_digest(DIG[name]))
    for a in ("i", "j", "k", "level", "values"):
        assert sha(getattr(cl, a)) == DIG[name][f"cells.{a}"], a


def test_validate_cells_report():
    from paper_2009_03076_b200.model import CellList, validate_cells

    rep = validate_cells(CellList([0, 0], [0, 0], [0, 0], [0, 0], [1.0, 1.0]))
    assert rep.duplicates == [(0, 1)] and rep.overlaps == []
    rep = validate_cells(CellList([0, 0], [0, 0], [0, 0], [0, 1], [1.0, 2.0]))
    assert rep.overlaps == [(0, 1)]
    rep = validate_cells(CellList([1], [0], [0], [1], [1.0]))
    assert rep.alignment == [0] and not rep.ok


def test_exacells_roundtrip_and_truncation(tmp_path):
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.model import CellList

    rng = np.random.default_rng(1)
    n = 300
    anchors = rng.choice(4096, n, replace=False)
    cl = CellList((anchors % 16) * 4 - 32, (anchors // 16 % 16) * 4, (anchors // 256) * 4, rng.integers(0, 3, n),
                  rng.random((n, 2), np.float32), ("a", "b"))
    p = tmp_path / "rt.exacells"
    xio.save_cells(p, cl)
    back = xio.load_cells(p)
    assert back.field_names == cl.field_names
    for a in ("i", "j", "k", "level", "values"):
        assert np.array_equal(getattr(back, a), getattr(cl, a))
    data = p.read_bytes()
    for cut in (1, 3, 4, 7, 8, 11, 15, 20, len(data) // 2, len(data) - 1):
        q = tmp_path / "cut.exacells"
        q.write_bytes(data[:cut])
        with pytest.raises(xio.ExaCellsError):
            xio.load_cells(q)


def test_artifact_roundtrip(tmp_path):
    from conftest import golden_model
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.model import AmrModel
    from paper_2009_03076_b200.regions import RegionSet

    g = golden_model("gauss16")
    m = AmrModel(("value",), g["model_brick_lower"], g["model_brick_level"], g["model_brick_dims"], g["model_scalars"])
    r = RegionSet(*(g[f"regions_{k}"] for k in ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")),
                  ("value",))
    xio.save_artifact(tmp_path / "a.npz", m, r)
    m2, r2, t2 = xio.load_artifact(tmp_path / "a.npz")
    assert t2 is None
    for k in ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars"):
        assert np.array_equal(getattr(m2, k), getattr(m, k))
    for k in ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width"):
        assert np.array_equal(getattr(r2, k), getattr(r, k))


def test_model_cell_list_canonical_order():
    from conftest import golden_model
    from paper_2009_03076_b200.model import AmrModel
    from tests_util import canonical_cells

    g = golden_model("smoke")
    m = AmrModel(("value",), g["model_brick_lower"], g["model_brick_level"], g["model_brick_dims"], g["model_scalars"])
    cl = m.cell_list()
    want = canonical_cells({k: g[f"model_{k}"] for k in ("brick_lower", "brick_level", "brick_dims", "brick_offset",
                                                          "scalars")})
    for a, w in zip((cl.i, cl.j, cl.k, cl.level), want[:4]):
        assert np.array_equal(a, w)


# ------------------------------------------------------------------ multi-GPU tiling (host logic)


@pytest.mark.parametrize("W,H,world", [(1024, 1024, 1), (1920, 1080, 2), (1920, 1080, 8), (97, 45, 3), (5, 3, 4)])
def test_tiles_partition_every_pixel_once(W, H, world):
    from paper_2009_03076_b200.parallel import packed_pixel_coords

    seen = np.zeros((H, W), np.int32)
    for r in range(world):
        x, y, valid = packed_pixel_coords(W, H, r, world)
        np.add.at(seen, (y[valid], x[valid]), 1)
    assert (seen == 1).all()


def test_parallel_generator_equals_serial():
    """generate_synthetic(workers=N) splits the frontier into chunks: same arrays, same order."""
    from paper_2009_03076_b200 import io as xio

    spec = xio.SyntheticSpec(field="gaussian", extent=(16384, 8192, 8192), max_level=12, threshold=0.05, seed=0,
                             holes=((6144.0, 6144.0, 6144.0, 40.0),), refine_spheres=((6144.0, 6144.0, 6144.0, 90.0),),
                             field_params={"center": (6144.0, 6144.0, 6144.0), "sigma": 600.0})
    a = xio.generate_synthetic(spec)
    b = xio.generate_synthetic(spec, workers=4)
    assert len(a) > (1 << 16)
    for k in ("i", "j", "k", "level", "values"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_scale_digest_fixture_pins_c2_cells():
    """tests/golden/scale_digests.json was made from the numpy generator's cells (the C2 entry is cheap to redo)."""
    import json
    import sys

    from tests_util import sha

    sys.path.insert(0, str(ROOT))
    import bench

    d = json.loads((ROOT / "tests" / "golden" / "scale_digests.json").read_text())
    assert {"c2", "c3"} <= set(d)
    cells = bench.make_cells(bench.CONFIGS["c2"])
    assert len(cells) == d["c2"]["n_cells"]
    for a in ("i", "j", "k", "level", "values"):
        assert sha(getattr(cells, a)) == d["c2"]["cells"][a], a
