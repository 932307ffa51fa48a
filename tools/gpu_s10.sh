#!/usr/bin/env bash
# Round-2 final measurement set I (final kernels and defaults): parity suite, smoke, every BASELINE
# configuration, default bench line with the CPU baseline.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 1500 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench cfg5 rc=$?" >> gpurun_out/status.txt
for c in cfg1 cfg2 cfg3 cfg5s cfg4; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
echo done >> gpurun_out/status.txt
