#!/usr/bin/env bash
# Round-2 measurement set N: ncu --set full of the HBM-bound level-13 target sums and of the split
# of configs[4] (seg_small / seg_gemm3 with the C-tile prefetch), arena capped at 80 GB.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export H2B_NVTX=1
export H2B_ARENA_GB=80
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "L13.targets:seg_gemm]" \
    -c 10 -o gpurun_out/l13_cfg5 -f python tools/one_product.py cfg5 > gpurun_out/ncu_l13_cfg5.log 2>&1
echo "ncu L13 cfg5 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh l13_cfg5 >> gpurun_out/status.txt 2>&1
echo done >> gpurun_out/status.txt
