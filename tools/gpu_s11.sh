#!/usr/bin/env bash
# Round-2 measurement set J: configs[3] at 64^3 with the default bench flags after the
# restore-in-place fix (8 consecutive products), parity subset, Gram tile choice for real products.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
H2B_MEM_TRACE=1 timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$?" >> gpurun_out/status.txt
grep -v "^\[mem\] L\|^\[mem\] leaf\|^\[mem\] basis\|^\[mem\] split" gpurun_out/bench_cfg4.err | tail -60 > gpurun_out/bench_cfg4.err.tail; rm -f gpurun_out/bench_cfg4.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ref_golden.py -x -q -m gpu -k "matches_oracle or golden or cfg4_like or nonleaf" > gpurun_out/t_parity.txt 2>&1; echo "parity rc=$?" >> gpurun_out/status.txt
for c in cfg2 cfg3; do
  for v in 0.75 0.9 1.0; do
    H2B_SYM_EFF32=$v timeout 1500 python bench.py --config $c --steps 4 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_eff$v.json 2> gpurun_out/bench_${c}_eff$v.err; echo "bench $c eff$v rc=$?" >> gpurun_out/status.txt
  done
done
echo done >> gpurun_out/status.txt
