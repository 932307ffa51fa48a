#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "truncation or small_tile" > gpurun_out/t_heev.txt 2>&1
echo "heev tests rc=$?" >> gpurun_out/status.txt
for cfg in cfg2 cfg5; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/b_${cfg}.json 2> gpurun_out/b_${cfg}.err
  echo "b_$cfg rc=$?" >> gpurun_out/status.txt
  H2B_EIG_LIBRARY=1 timeout 900 python bench.py --config $cfg --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/bl_${cfg}.json 2> gpurun_out/bl_${cfg}.err
  echo "bl_$cfg rc=$?" >> gpurun_out/status.txt
done
