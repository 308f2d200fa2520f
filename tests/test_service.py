"""Render service on GPU scenes (R/service.py): the
shared Session's snapshot semantics and the websocket frame protocol, with the
reference's test cases restated (T/test_service.py) plus the raw encoding."""
import io
import json
import threading

import numpy as np
import pytest

from tests_util import golden_cells

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks
    from paper_2009_03076_b200.model import CellList
    from paper_2009_03076_b200.regions import build_regions

    i, j, k, lev, vals = golden_cells("smoke")
    model, tree = build_bricks(CellList(i, j, k, lev, vals), BrickBuildParams(keep_split_tree=True))
    return model, build_regions(model), tree


def _ramp(lo, hi, alpha):
    rgba = np.zeros((256, 4))
    rgba[:, 0] = rgba[:, 1] = rgba[:, 2] = np.linspace(0, 1, 256)
    rgba[:, 3] = np.linspace(0, alpha, 256)
    return {"domain": [lo, hi], "rgba": rgba.tolist()}


def test_session_edits_snapshot_and_rebuild_accounting(built):
    from paper_2009_03076_b200.render import render_frame
    from paper_2009_03076_b200.service import ProtocolError, Session

    model, regions, tree = built
    s = Session(model, regions, tree)
    info = s.info()
    assert info["stats"]["regions"] == len(regions) and info["stats"]["hasTree"]
    fid, f0 = s.render(64, 48)
    assert fid == 1 and f0.stats.bvh_rebuild_ms == 0.0 and f0.stats.samples > 0
    lo, hi = model.value_range(0)
    old_scene = s.scene
    s.set_tf(_ramp(lo, hi, 0.2))
    assert s.scene is not old_scene and old_scene.volume_bvh is not s.scene.volume_bvh  # fresh snapshot
    s.set_iso({"value": float(0.5 * (lo + hi))})
    fid, f1 = s.render(64, 48)
    assert fid == 2 and f1.stats.bvh_rebuild_ms > 0.0
    _, f2 = s.render(64, 48)
    assert f2.stats.bvh_rebuild_ms == 0.0  # reported once
    # the snapshot renders exactly like render_frame on the same scene
    from paper_2009_03076_b200.render import Camera

    c = s._snap.camera
    cam = Camera(c["pos"], np.asarray(c["look"]) - np.asarray(c["pos"]), c["up"], c["fov"], 64, 48)
    assert np.array_equal(render_frame(s.scene, cam, s._snap.tf, s._snap.params).rgba, f2.rgba)
    s.set_iso({"value": None})
    assert s.scene.iso_bvh is None
    for bad in ({"domain": [1, 0], "rgba": [[0, 0, 0, 0]] * 256}, {"domain": [0, 1]}):
        with pytest.raises(ProtocolError):
            s.set_tf(bad)
    with pytest.raises(ProtocolError):
        s.set_params({"gradientMode": "nope"})
    with pytest.raises(ProtocolError):
        s.set_camera({"fov": 200})


def test_concurrent_renders_are_consistent(built):
    from paper_2009_03076_b200.service import Session

    model, regions, tree = built
    s = Session(model, regions, tree)
    _, ref = s.render(80, 60)
    out, errs = [], []

    def worker():
        try:
            for _ in range(3):
                out.append(s.render(80, 60)[1].rgba)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=worker) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs and len(out) == 12 and all(np.array_equal(o, ref.rgba) for o in out)


def test_websocket_protocol(built):
    from fastapi.testclient import TestClient
    from PIL import Image

    from paper_2009_03076_b200.service import make_app

    model, regions, tree = built
    app = make_app(model, regions, tree)
    client = TestClient(app)
    assert client.get("/health").json()["status"] == "ok"
    with client.websocket_connect("/ws") as ws:
        ws.send_text(json.dumps({"type": "hello"}))
        assert json.loads(ws.receive_text())["type"] == "info"
        ws.send_text(json.dumps({"type": "set_params", "seed": 7, "gradientMode": "analytic"}))
        frames = {}
        for enc in ("png", "raw", "png-fast"):
            ws.send_text(json.dumps({"type": "request_frame", "width": 40, "height": 30, "encoding": enc}))
            hdr = json.loads(ws.receive_text())
            body = ws.receive_bytes()
            assert hdr["type"] == "frame" and hdr["encoding"] == enc and hdr["stats"]["samples"] > 0
            if enc == "raw":
                frames[enc] = np.frombuffer(body, np.uint8).reshape(30, 40, 4)
            else:
                frames[enc] = np.asarray(Image.open(io.BytesIO(body)).convert("RGBA"))
        assert np.array_equal(frames["png"], frames["raw"]) and np.array_equal(frames["png-fast"], frames["raw"])
        for bad, code in ((b"not json", "bad_json"), (json.dumps([1]).encode(), "bad_json"),
                          (json.dumps({"type": "bogus"}).encode(), "unsupported"),
                          (json.dumps({"type": "request_frame", "width": 0}).encode(), "bad_message"),
                          (json.dumps({"type": "request_frame", "encoding": "jpeg"}).encode(), "bad_message")):
            ws.send_text(bad.decode())
            err = json.loads(ws.receive_text())
            assert err["type"] == "error" and err["code"] == code


def test_concurrent_mixed_renders_and_tf_edits(built):
    """8 threads render different views, sizes, gradient modes and iso settings of
    one model concurrently (the reference renders outside its lock,
    R/service.py:166-176) while another thread keeps rebuilding active sets for
    new TFs; every frame must equal its sequential render."""
    from paper_2009_03076_b200.accel import TransferFunction, build_volume_bvh
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame

    model, regions, tree = built
    lo, hi = model.value_range(0)
    tf = TransferFunction.grayscale((lo, hi), max_alpha=0.6)
    scenes = [build_scene(model, regions, tf), build_scene(model, regions, tf, iso_value=0.5 * (lo + hi))]
    jobs = []
    for k, (w, h) in enumerate([(64, 48), (96, 64), (40, 40), (128, 72)]):
        for v, cam in enumerate(orbit_cameras(regions.bounds, 4, w, h)):
            gm = ("analytic", "central", "none")[(k + v) % 3]
            jobs.append((scenes[(k + v) % 2], cam, MarchParams(seed=k + v, gradient_mode=gm)))
    ref = [render_frame(sc, cam, tf, p) for sc, cam, p in jobs]
    errs, results = [], {}
    stop = threading.Event()

    def editor():
        try:
            a = 0.1
            while not stop.is_set():
                build_volume_bvh(regions, TransferFunction.grayscale((lo, hi), max_alpha=a), 0, model=model)
                a = 0.1 + (a + 0.13) % 0.8
        except Exception as e:  # pragma: no cover
            errs.append(e)

    def worker(t):
        try:
            for rep in range(3):
                for q in range(t, len(jobs), 8):
                    sc, cam, p = jobs[q]
                    results[(q, rep)] = render_frame(sc, cam, tf, p)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ed = threading.Thread(target=editor)
    ed.start()
    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    stop.set()
    ed.join()
    assert not errs, errs
    assert len(results) == 3 * len(jobs)
    for (q, rep), fr in results.items():
        assert np.array_equal(fr.rgba, ref[q].rgba), (q, rep)
        assert (fr.stats.regions, fr.stats.samples) == (ref[q].stats.regions, ref[q].stats.samples)
