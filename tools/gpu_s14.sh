#!/usr/bin/env bash
# Round-2 measurement set M: the reference arm (the reference's own mmp(), 1 thread) on the other BASELINE configurations.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3; do
  timeout 900 python bench.py --impl reference --config $c --steps 5 --warmup 3 > gpurun_out/bench_reference_$c.json 2> gpurun_out/bench_reference_$c.err; echo "reference $c rc=$?" >> gpurun_out/status.txt
done
echo done >> gpurun_out/status.txt
