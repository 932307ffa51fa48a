#!/usr/bin/env bash
# Round-2 measurement set H: A/B of the seg_small chunk bound for complex products and of the
# Hermitian (Gram) tile choice, on the configs[4] construction at 2^18 and at 2^20.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in cfg5s cfg5; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_default.json 2> gpurun_out/bench_${c}_default.err; echo "bench $c default rc=$?" >> gpurun_out/status.txt
  for v in 8 24 64; do
    H2B_SMALL_MAXCH=$v timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_maxch$v.json 2> gpurun_out/bench_${c}_maxch$v.err; echo "bench $c maxch$v rc=$?" >> gpurun_out/status.txt
  done
  for v in 0.76 1.0; do
    H2B_SYM_EFF32=$v timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_eff$v.json 2> gpurun_out/bench_${c}_eff$v.err; echo "bench $c eff$v rc=$?" >> gpurun_out/status.txt
  done
done
echo done >> gpurun_out/status.txt
