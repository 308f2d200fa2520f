"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_digests():
    with open(GOLDEN / "digests.json") as fh:
        return json.load(fh)


def golden_model(name):
    return dict(np.load(GOLDEN / f"model_{name}.npz"))


def golden_frames():
    """frames.npz (make_golden.py) + frames_inside.npz (make_inside.py: eyes inside the volume)."""
    fr = dict(np.load(GOLDEN / "frames.npz"))
    fr.update(np.load(GOLDEN / "frames_inside.npz"))
    return fr


def frame_meta(frames, key):
    return json.loads(bytes(frames[f"{key}_meta"]).decode())


@pytest.fixture(scope="session")
def digests():
    return golden_digests()


@pytest.fixture(scope="session")
def frames():
    return golden_frames()
