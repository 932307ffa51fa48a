#!/bin/bash
# heev placement sweep on the Gram sizes / counts of configs[1]'s levels (row + column launches of a
# level run concurrently: count = 2 x clusters) and configs[4]'s upper levels (complex).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for spec in "624 32 0" "576 64 0" "512 128 0" "416 256 0" "256 512 0" "456 64 1" "344 128 1" "240 256 1" "184 512 1"; do
  set -- $spec
  for mode in "1 0" "2 0" "4 0" "8 0" "16 0" "4 1" "8 1" "16 1"; do
    set -- $spec $mode
    timeout 120 tools/heev_bench $1 $2 $3 0 512 $4 $5 2>&1 | grep "^heev\|CUDA"
  done
done
} > gpurun_out/heev_sweep.txt 2>&1
echo "heev sweep rc=$?" >> gpurun_out/status.txt
