"""GPU synthetic generator (csrc/synth.cu) against the reference's own
generator output (sha256 digests of R/io.py:generate_synthetic, produced by
tests/golden/make_golden.py) and against the package's numpy restatement at
scale; device-resident cells through build_bricks."""
import numpy as np
import pytest

from conftest import golden_digests
from tests_util import sha, spec_from_digest

pytestmark = pytest.mark.gpu

DIG = golden_digests()["models"]
SPEC_NAMES = sorted(n for n, d in DIG.items() if "spec" in d)


def _ulps32(a, b):
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return np.abs(ia - ib)


@pytest.mark.parametrize("name", SPEC_NAMES)
def test_device_generator_matches_reference_digests(name):
    from paper_2009_03076_b200 import io as xio

    spec = spec_from_digest(DIG[name])
    dc = xio.generate_synthetic_device(spec)
    cl = dc.to_host()
    assert len(cl) == DIG[name]["n_cells"]
    for a in ("i", "j", "k", "level"):
        assert sha(getattr(cl, a)) == DIG[name][f"cells.{a}"], f"{name}: cells.{a}"
    if sha(cl.values) != DIG[name]["cells.values"]:
        # CUDA's exp/sin vs numpy's: allowed only as isolated 1-ulp float32 roundings
        host = xio.generate_synthetic(spec)  # pinned to the same digest by test_host.py
        assert sha(host.values) == DIG[name]["cells.values"]
        u = _ulps32(cl.values[:, 0], host.values[:, 0])
        assert u.max() <= 1 and np.count_nonzero(u) <= max(1, len(cl) // 100000), (name, u.max(), np.count_nonzero(u))


def test_device_generator_c2_scale_matches_host():
    """configs[1] (9.53M cells): every cell identical to the numpy generator."""
    from paper_2009_03076_b200 import io as xio

    spec = xio.SyntheticSpec(field="gaussian", extent=(256, 256, 256), max_level=3, threshold=0.004, seed=0)
    dev = xio.generate_synthetic_device(spec).to_host()
    host = xio.generate_synthetic(spec)
    assert len(dev) == len(host) == 9_534_568
    for a in ("i", "j", "k", "level"):
        assert np.array_equal(getattr(dev, a), getattr(host, a)), a
    u = _ulps32(dev.values[:, 0], host.values[:, 0])
    assert u.max() <= 1 and np.count_nonzero(u) <= 100, (u.max(), np.count_nonzero(u))


def test_build_bricks_from_device_cells_equals_host_path():
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks

    spec = spec_from_digest(DIG["smoke"])
    dc = xio.generate_synthetic_device(spec)
    m_dev, t_dev = build_bricks(dc, BrickBuildParams(keep_split_tree=True))
    m_host, t_host = build_bricks(dc.to_host(), BrickBuildParams(keep_split_tree=True))
    for k in ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars"):
        assert np.array_equal(getattr(m_dev, k), getattr(m_host, k)), k
    for k in ("axis", "pos", "left", "right", "brick_start", "brick_count"):
        assert np.array_equal(getattr(t_dev, k), getattr(t_host, k)), k


def test_landing_gear_shape_generates_all_levels():
    """A 1/4-scale Landing-Gear-shaped spec (SURVEY.md §8(d) C3 template): 12
    refinement steps, a hole, a level-0 shell; deterministic across runs."""
    from paper_2009_03076_b200 import io as xio

    spec = xio.SyntheticSpec(field="gaussian", extent=(16384, 8192, 8192), max_level=12, threshold=0.05, seed=0,
                             holes=((6144, 6144, 6144, 60.0),), refine_spheres=((6144, 6144, 6144, 130.0),),
                             field_params={"center": (6144.0, 6144.0, 6144.0), "sigma": 600.0})
    a = xio.generate_synthetic_device(spec).to_host()
    b = xio.generate_synthetic_device(spec).to_host()
    assert np.array_equal(a.i, b.i) and np.array_equal(a.values, b.values)
    lv = np.bincount(a.level, minlength=13)
    assert lv[0] > 4_000_000 and lv[12] > 0 and lv.sum() == len(a), lv
    c = np.stack([a.i, a.j, a.k], 1).astype(np.float64) + (2.0 ** a.level)[:, None] / 2
    assert not np.any(np.sum((c - 6144.0) ** 2, axis=1) < 60.0 ** 2)  # the hole is empty


def test_streamed_exacells_loader(tmp_path):
    """io.load_cells_device streams a .exacells file to the GPU in chunks
    (R/io.py:88-113 format): same cells as load_cells, same bricks."""
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.bricks import build_bricks

    cl = xio.generate_synthetic(spec_from_digest(DIG["gauss_aniso"]))
    path = tmp_path / "m.exacells"
    xio.save_cells(path, cl)
    for chunk in (1000, 1 << 24):  # many chunks / one chunk
        dc = xio.load_cells_device(path, chunk=chunk)
        back = dc.to_host()
        for a in ("i", "j", "k", "level", "values"):
            assert np.array_equal(getattr(back, a), getattr(cl, a)), (chunk, a)
    m_dev, _ = build_bricks(dc)
    m_host, _ = build_bricks(cl)
    for k in ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars"):
        assert np.array_equal(getattr(m_dev, k), getattr(m_host, k)), k
    with open(path, "ab") as fh:
        fh.write(b"x")
    with pytest.raises(xio.ExaCellsError):
        xio.load_cells_device(path)
