#!/usr/bin/env bash
# One measurement round on a B200 (run under gpurun from the repo root):
#   1. GPU parity tests           -> gpurun_out/pytest_gpu.log
#   2. bench line (configs[1])    -> gpurun_out/bench_<cfg>.json
#   3. ncu launch list of one product of the bench workload, kernels renamed by their NVTX phase
#                                 -> gpurun_out/launches_<cfg>.csv
#   4. ncu --set full of the dominant phase's kernel (NVTX-selected)
#                                 -> gpurun_out/top_<cfg>.ncu-rep
# Usage: bash tools/gpu_round.sh [cfg] [phase-range] [skip-tests]
set -u
CFG=${1:-cfg2}
RANGE=${2:-L9.targets:seg_gemm}
SKIP_TESTS=${3:-0}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
if [ "$SKIP_TESTS" = "0" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --config "$CFG" --steps 5 --warmup 3 --profile > gpurun_out/bench_${CFG}.json 2> gpurun_out/bench_${CFG}.err
echo "bench exit $?"
NCU=/usr/local/cuda/bin/ncu
export H2B_NVTX=1
CMD="python tools/one_product.py $CFG"
timeout 600 $CMD > gpurun_out/plain_${CFG}.log 2>&1 &&
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename kernel \
    --csv --log-file gpurun_out/launches_${CFG}.csv $CMD > gpurun_out/ncu_launches_${CFG}.log 2>&1
echo "launch list exit $?"
timeout 600 python tools/one_product.py "$CFG" > gpurun_out/plain_repro_${CFG}.log 2>&1 &&
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "${RANGE}]" -c 8 \
    -o gpurun_out/top_${CFG} -f python tools/one_product.py "$CFG" > gpurun_out/ncu_full_${CFG}.log 2>&1
echo "ncu full exit $?"
