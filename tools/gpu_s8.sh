#!/usr/bin/env bash
# Round-2 measurement set G: heev global-slab passes with 8 (was 4) loads in flight per lane:
# standalone A/B, parity suite, benches, final default bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for spec in "624 32 0 4" "576 64 0 2" "512 128 0 1" "416 256 0 1" "256 512 0 1" "464 16 0 4" "456 64 1 2" "344 128 1 1" "240 256 1 1" "344 32 1 4"; do
  set -- $spec
  for B in tools/heev_bench_u4 tools/heev_bench; do
    echo -n "$B: "; timeout 120 $B $1 $2 $3 0 512 $4 0 2>&1 | grep "^heev\|CUDA"
  done
done
} > gpurun_out/heev_u8.txt 2>&1
echo "heev A/B rc=$?" >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for c in cfg2 cfg5s cfg3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
timeout 1500 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench cfg5 rc=$?" >> gpurun_out/status.txt
echo done >> gpurun_out/status.txt
