cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "acceptance or frames_match" > gpurun_out/pt_fac.log 2>&1; tail -2 gpurun_out/pt_fac.log
timeout 300 python tools/ab.py c2 warp 6 > gpurun_out/ab_fac.log 2>&1; grep median gpurun_out/ab_fac.log
XB_LIB=$PWD/paper_2009_03076_b200/libexabricks_exact.so timeout 300 python tools/ab.py c2 warp 6 > gpurun_out/ab_facx.log 2>&1; grep median gpurun_out/ab_facx.log
timeout 300 python tools/ab.py c3 warp 6 > gpurun_out/ab_fac3.log 2>&1; grep median gpurun_out/ab_fac3.log
XB_LIB=$PWD/paper_2009_03076_b200/libexabricks_exact.so timeout 300 python tools/ab.py c3 warp 6 > gpurun_out/ab_facx3.log 2>&1; grep median gpurun_out/ab_facx3.log
