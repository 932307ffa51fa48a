#!/usr/bin/env bash
# Round-2 measurement set D (what the driver runs at round end, plus the arena-cap check):
# full parity suite, smoke, default bench (configs[4]) with the CPU baseline, the reference arm,
# configs[4] under a capped arena (eviction path).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
( time timeout 1500 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err ) 2> gpurun_out/bench_cfg5.time; echo "bench cfg5 rc=$?" >> gpurun_out/status.txt
( time timeout 1800 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err ) 2> gpurun_out/bench_reference.time; echo "bench reference rc=$?" >> gpurun_out/status.txt
H2B_ARENA_GB=80 H2B_MEM_TRACE=1 timeout 600 python -X faulthandler tools/one_product.py cfg5 > gpurun_out/arena80_cfg5.out 2> gpurun_out/arena80_cfg5.err; echo "arena80 cfg5 rc=$?" >> gpurun_out/status.txt
tail -c 6000 gpurun_out/arena80_cfg5.err > gpurun_out/arena80_cfg5.err.tail; rm -f gpurun_out/arena80_cfg5.err
for c in cfg3 cfg5s; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/shape_profile.py cfg3 60 > gpurun_out/shapes_cfg3.txt 2>&1
echo done >> gpurun_out/status.txt
du -sh gpurun_out >> gpurun_out/status.txt
