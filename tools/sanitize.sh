# usage: gpurun -- bash tools/sanitize.sh TAG   -> gpurun_out/sanitize_{memcheck,racecheck,synccheck}_TAG.log
cd "${GRAFT_REPO_ROOT:-.}"; TAG=${1:-v}; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_frames.py \
    > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}_$TAG.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/sanitize_smoke_$TAG.log 2>&1; echo "smoke memcheck rc=$?"; tail -3 gpurun_out/sanitize_smoke_$TAG.log
