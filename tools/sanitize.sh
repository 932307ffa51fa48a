#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py, one tool per call: bash tools/sanitize.sh memcheck|racecheck|synccheck
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${1:-memcheck}
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$T.txt 2>&1
echo "sanitize $T rc=$?" >> gpurun_out/status.txt
