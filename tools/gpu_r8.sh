#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matches_oracle or cfg1 or nonleaf or complex or truncation" > gpurun_out/t_parity.txt 2>&1
echo "parity rc=$?" >> gpurun_out/status.txt
{
for a in "128 512 0" "406 128 0" "566 32 0" "610 16 0" "64 2048 1" "104 512 1" "216 64 1" "600 8 1"; do
  set -- $a
  timeout 120 tools/heev_bench5 $1 $2 $3 0
  timeout 120 tools/heev_bench5 $1 $2 $3 0 512 1 0
done
} > gpurun_out/heev_v5.txt 2>&1
H2B_MEM_TRACE=1 timeout 1500 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
echo "b_cfg4 rc=$?" >> gpurun_out/status.txt
for cfg in cfg2 cfg5; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err
echo "b_$cfg rc=$?" >> gpurun_out/status.txt
done
