#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B=tools/heev_bench
{
for a in "128 512 0" "256 256 0" "406 128 0" "504 64 0" "566 32 0" "610 16 0" "556 8 0" "450 4 0" "390 2 0" \
         "40 8192 1" "48 4096 1" "64 2048 1" "80 1024 1" "104 512 1" "128 256 1" "160 128 1" "216 64 1" "320 32 1" "450 16 1" "600 8 1" "700 4 1"; do
  set -- $a
  timeout 120 $B $1 $2 $3 0 | grep heev
  timeout 120 $B $1 $2 $3 0 512 1 0 | grep heev
done
} > gpurun_out/heev_shapes.txt 2>&1
echo "shapes done" >> gpurun_out/status.txt
H2B_MEM_TRACE=1 timeout 1200 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
echo "b_cfg4 rc=$?" >> gpurun_out/status.txt
