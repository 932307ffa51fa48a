#!/usr/bin/env bash
# Round-2 measurement set K: eviction with deferred in-place operand restore: configs[3] at 64^3 with
# the default bench flags (9 consecutive products), configs[4] under an 80 GB arena, parity subset.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
H2B_MEM_TRACE=1 timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$?" >> gpurun_out/status.txt
grep "evicted\|L11.targets\|Error\|error\|Traceback" gpurun_out/bench_cfg4.err | tail -80 > gpurun_out/bench_cfg4.err.tail; rm -f gpurun_out/bench_cfg4.err
H2B_ARENA_GB=80 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_cfg5_arena80.json 2> gpurun_out/bench_cfg5_arena80.err; echo "bench cfg5 arena80 rc=$?" >> gpurun_out/status.txt
tail -c 3000 gpurun_out/bench_cfg5_arena80.err > gpurun_out/bench_cfg5_arena80.err.tail; rm -f gpurun_out/bench_cfg5_arena80.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ref_golden.py tests/test_dropin_cpp.py -x -q -m gpu -k "matches_oracle or golden or cfg4_like or dropin or mvp or dense" > gpurun_out/t_parity.txt 2>&1; echo "parity rc=$?" >> gpurun_out/status.txt
echo done >> gpurun_out/status.txt
