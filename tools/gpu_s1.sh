#!/usr/bin/env bash
# Round-2 measurement set A on one B200 (under gpurun): parity suite, default bench (configs[4]),
# launch list and ncu --set full of the dominant kernel of the same workload, other configs.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 1200 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench cfg5 rc=$?" >> gpurun_out/status.txt
export H2B_NVTX=1
timeout 900 python tools/one_product.py cfg5 > gpurun_out/plain_one_cfg5.log 2>&1 &&
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename kernel \
    --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_product.py cfg5 > gpurun_out/ncu_launches_cfg5.log 2>&1
echo "launch list rc=$?" >> gpurun_out/status.txt
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    -c 2 -o gpurun_out/top_cfg5 -f python tools/one_product.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/status.txt
unset H2B_NVTX
for c in cfg2 cfg3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/shape_profile.py cfg3 30 > gpurun_out/shapes_cfg3.txt 2>&1
echo done >> gpurun_out/status.txt
