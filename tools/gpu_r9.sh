#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "matches_oracle or nonleaf or cfg5_like or cfg3_like or cfg4_like" > gpurun_out/t_parity.txt 2>&1
echo "parity rc=$?" >> gpurun_out/status.txt
H2B_MEM_TRACE=1 timeout 1500 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
echo "b_cfg4 rc=$?" >> gpurun_out/status.txt
