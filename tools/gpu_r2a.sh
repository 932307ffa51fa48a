#!/usr/bin/env bash
# Round-2 measurement pass on one B200 (run under gpurun from the repo root).
set -u
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
s=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $? $(( $(date +%s)-s )) s" >> gpurun_out/status.txt
s=$(date +%s)
timeout 1200 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench exit $? $(( $(date +%s)-s )) s" >> gpurun_out/status.txt
s=$(date +%s)
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $? $(( $(date +%s)-s )) s" >> gpurun_out/status.txt
export H2B_NVTX=1
timeout 900 python tools/one_product.py cfg5 > gpurun_out/plain_one_cfg5.log 2>&1 &&
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename kernel \
    --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_product.py cfg5 > gpurun_out/ncu_launches_cfg5.log 2>&1
echo "launches exit $?" >> gpurun_out/status.txt
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    --kernel-name-base demangled -k "regex:seg_gemm3_kernel<\(int\)64, \(int\)64" -c 1 -o gpurun_out/top_cfg5 -f \
    python tools/one_product.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo "ncu full exit $?" >> gpurun_out/status.txt
