"""bench.py's JSON line keeps the driver's contract (keys, types, units) —
run on the small configs[0] workload so it finishes in seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_contract():
    d = _run("--config", "c1", "--secondary", "", "--extra", "", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "frames/s" and d["dtype"] == "f64"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s"
    assert 0 < r["achieved"] and 0 < r["peak"] and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] >= 4 * 256 * 256
    assert d["gpu_launches"] >= 5 * d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # parity measured in the run: the oracle's bands of orbit view 0 against the GPU frame
    p = d["parity"]
    assert p["ok"] is True and p["frame"]["max_abs_drgba"] <= 1e-3
    assert p["frame"]["px_region_counter_mismatches"] == 0 and p["frame"]["px_sample_counter_mismatches"] == 0
    assert len(d["views"]) == d["config"]["views"] == 8
    assert r["kernel"].startswith("k_warp") and r["frame_achieved"] <= r["achieved"]


@pytest.mark.gpu
def test_bench_reference_arm_contract():
    d = _run("--impl", "reference", "--config", "c1", "--secondary", "", "--extra", "", "--steps", "1",
             "--warmup", "1", "--cpu-seconds", "1")
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "frames/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    ours = _run("--config", "c1", "--secondary", "", "--extra", "", "--steps", "1", "--warmup", "1",
                "--no-cpu-baseline", "--no-ablations")
    assert d["config"] == ours["config"]  # same workload, same keys: the driver's same_config


def test_reference_arm_loads_no_gpu_library():
    """The reference arm runs host code only: libexabricks.so is never mapped."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
            "'--warmup','1']; import bench; bench.main(sys.argv[1:]);"
            "maps=open('/proc/self/maps').read(); print('LIB', 'libexabricks' in maps)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "LIB False" in out.stdout


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu():
    """The N > 1 path of bench.py end to end on a one-GPU box: `--gpus 2`
    relaunches under torch.distributed.run, both ranks share cuda:0 over gloo
    (XB_BENCH_SHARE_GPU=1; NCCL refuses two ranks on one device), cells are
    broadcast from rank 0, tiles rendered per rank, gathered, unpacked and the
    counters all-reduced: the frame counters equal the one-rank run's."""
    env = dict(os.environ, XB_BENCH_SHARE_GPU="1")
    args = ["--config", "c1", "--secondary", "", "--extra", "", "--steps", "2", "--warmup", "1"]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", *args], capture_output=True,
                         text=True, cwd=ROOT, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d2 = json.loads(lines[0])
    d1 = _run(*args, "--no-cpu-baseline")
    assert d2["n_gpus"] == 2 and d2["nccl"]["world"] == 2 and d2["value"] > 0
    assert d2["frame"] == d1["frame"]  # counters of the tiled frame, summed over the ranks
    assert d2["e2e"]["value"] > 0
