cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
python tools/e2e_probe.py c3 30 2>&1 | tail -8
XB_BANDS=0 python tools/e2e_probe.py c3 30 2>&1 | grep -E "render_frame|pinned"
