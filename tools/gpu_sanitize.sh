# compute-sanitizer over tools/sanitize_case.py, ONE tool per gpurun call:
#   bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck
TOOL=${1:-memcheck}
python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 3000 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitize $TOOL rc=$?"; tail -5 gpurun_out/sanitize_$TOOL.log
