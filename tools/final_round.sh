#!/usr/bin/env bash
# Round-end measurement set on one B200 (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in cfg3 cfg5s cfg4s; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 1500 python bench.py --config cfg5 --steps 3 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 300 python tools/shape_profile.py cfg3 30 > gpurun_out/shapes_cfg3.txt 2>&1
export H2B_NVTX=1
timeout 600 python tools/one_product.py cfg2 > gpurun_out/plain_one_cfg2.log 2>&1 &&
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename kernel \
    --csv --log-file gpurun_out/launches_cfg2.csv python tools/one_product.py cfg2 > gpurun_out/ncu_launches_cfg2.log 2>&1
timeout 900 python tools/one_product.py cfg5 > gpurun_out/plain_one_cfg5.log 2>&1 &&
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    --kernel-name-base demangled -k "regex:seg_gemm3_kernel<\(int\)64, \(int\)64" -c 1 -o gpurun_out/top_cfg5 -f \
    python tools/one_product.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo done
