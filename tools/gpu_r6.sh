#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for a in "128 512 0" "256 256 0" "406 128 0" "504 64 0" "566 32 0" "610 16 0" "64 2048 1" "80 1024 1" "104 512 1" "128 256 1" "216 64 1" "320 32 1" "600 8 1"; do
  set -- $a
  timeout 120 tools/heev_bench4 $1 $2 $3 0
  timeout 120 tools/heev_bench4 $1 $2 $3 0 512 1 0
done
} > gpurun_out/heev_v4.txt 2>&1
echo "v4 done" >> gpurun_out/status.txt
H2B_MEM_TRACE=1 timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
echo "b_cfg4 rc=$?" >> gpurun_out/status.txt
