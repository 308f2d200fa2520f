cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_service.py -q -m gpu -x --timeout 900 > gpurun_out/pt_svc1.log 2>&1; tail -25 gpurun_out/pt_svc1.log
