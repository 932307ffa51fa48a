#!/usr/bin/env bash
# Round-2 measurement set E: seg_small with the parallel index prologue, heev global slabs from 12
# Grams: parity suite, benches, heev check, the metric vs N, configs[3] at 64^3, launch list and
# ncu --set full of the dominant configs[4] kernel.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for c in cfg3 cfg5s cfg2 cfg1; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/shape_profile.py cfg3 60 > gpurun_out/shapes_cfg3.txt 2>&1
{
  for mode in "4 0" "8 0" "16 0" "16 1"; do set -- $mode; timeout 120 tools/heev_bench 464 16 0 0 512 $1 $2 2>&1 | grep "^heev\|CUDA"; done
  for mode in "8 0" "16 0" "16 1"; do set -- $mode; timeout 120 tools/heev_bench 392 8 0 0 512 $1 $2 2>&1 | grep "^heev\|CUDA"; done
  for mode in "4 0" "8 0" "16 1"; do set -- $mode; timeout 120 tools/heev_bench 344 32 1 0 512 $1 $2 2>&1 | grep "^heev\|CUDA"; done
} > gpurun_out/heev_sweep2.txt 2>&1
timeout 1500 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$?" >> gpurun_out/status.txt
timeout 2400 python tools/sweep_n.py gpurun_out/sweep_n.json > gpurun_out/sweep_n.log 2>&1; echo "sweep rc=$?" >> gpurun_out/status.txt
export H2B_NVTX=1
timeout 900 python tools/one_product.py cfg5 > gpurun_out/plain_one_cfg5.log 2>&1 &&
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename kernel \
    --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_product.py cfg5 > gpurun_out/ncu_launches_cfg5.log 2>&1
echo "launch list rc=$?" >> gpurun_out/status.txt
python tools/launch_summary.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5_summary.txt 2>&1
gzip -f gpurun_out/launches_cfg5.csv
export H2B_ARENA_GB=80
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    --kernel-name-base demangled -k "regex:seg_gemm3_kernel<(\(int\))?64, (\(int\))?64" -c 1 -o gpurun_out/top_cfg5 -f \
    python tools/one_product.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo "ncu full cfg5 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh top_cfg5 >> gpurun_out/status.txt 2>&1
echo done >> gpurun_out/status.txt
du -sh gpurun_out >> gpurun_out/status.txt
