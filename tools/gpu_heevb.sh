#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for B in tools/heev_bench tools/heev_bench_div; do
  for dbg in 0 1; do
    echo "== $B dbg=$dbg"
    timeout 120 $B 610 2 0 0 512 16 1 $dbg
    timeout 120 $B 406 16 0 0 512 8 1 $dbg
    timeout 120 $B 128 64 0 0 256 1 1 $dbg
  done
done
} > gpurun_out/heevb2.txt 2>&1
