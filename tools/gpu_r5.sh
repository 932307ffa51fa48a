#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for a in "128 512 0" "256 256 0" "406 128 0" "504 64 0" "566 32 0" "64 2048 1" "80 1024 1" "104 512 1" "128 256 1" "216 64 1" "600 8 1"; do
  set -- $a
  timeout 120 tools/heev_bench3 $1 $2 $3 0 | grep heev
  timeout 120 tools/heev_bench3 $1 $2 $3 0 512 1 0 | grep heev
done
} > gpurun_out/heev_v3.txt 2>&1
echo "v3 done" >> gpurun_out/status.txt
bash tools/gpu_fixtures.sh cfg3 cfg5s cfg2
