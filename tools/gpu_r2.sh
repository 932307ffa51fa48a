#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py -x -q -k "truncation or dropin or matches_oracle" > gpurun_out/t_a.txt 2>&1
echo "tests rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
echo "b_cfg2 rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err
echo "b_cfg5 rc=$?" >> gpurun_out/status.txt
H2B_MEM_TRACE=1 timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
echo "b_cfg4 rc=$?" >> gpurun_out/status.txt
timeout 1200 python tools/order_caps.py 1048576 5,7,9 > gpurun_out/caps.txt 2>&1
echo "caps rc=$?" >> gpurun_out/status.txt
