#!/usr/bin/env bash
# Round-2 measurement set B2: parity + bench of the index-prefetch seg_gemm3, ncu --set full of the
# HBM-bound / latency-bound kernels on configs[2] (small-rank target sums, heev, seg_add, gram_combine)
# and of the dominant kernel on the configs[4] construction at 2^18, heev placement sweep, memcheck.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size_fixtures.py -x -q -m gpu > gpurun_out/t_parity.txt 2>&1; echo "parity rc=$?" >> gpurun_out/status.txt
for c in cfg3 cfg5s cfg2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/shape_profile.py cfg3 40 > gpurun_out/shapes_cfg3.txt 2>&1
export H2B_NVTX=1
export H2B_ARENA_GB=40
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "L12.targets:seg_gemm]" \
    -c 8 -o gpurun_out/l12_cfg3 -f python tools/one_product.py cfg3 > gpurun_out/ncu_l12_cfg3.log 2>&1
echo "ncu L12 cfg3 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh l12_cfg3 >> gpurun_out/status.txt 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "regex:.*:heev]" \
    -c 4 -o gpurun_out/heev_cfg3 -f python tools/one_product.py cfg3 > gpurun_out/ncu_heev_cfg3.log 2>&1
echo "ncu heev cfg3 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh heev_cfg3 >> gpurun_out/status.txt 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "regex:.*:(seg_add|gram_combine)]" \
    -c 4 -o gpurun_out/hbm_cfg3 -f python tools/one_product.py cfg3 > gpurun_out/ncu_hbm_cfg3.log 2>&1
echo "ncu hbm cfg3 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh hbm_cfg3 >> gpurun_out/status.txt 2>&1
export H2B_ARENA_GB=70
timeout 1200 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    -c 1 -o gpurun_out/top_cfg5s -f python tools/one_product.py cfg5s > gpurun_out/ncu_full_cfg5s.log 2>&1
echo "ncu full cfg5s rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh top_cfg5s >> gpurun_out/status.txt 2>&1
unset H2B_NVTX H2B_ARENA_GB
bash tools/gpu_heev_sweep.sh
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_memcheck.txt 2>&1
echo "sanitize memcheck rc=$?" >> gpurun_out/status.txt
echo done >> gpurun_out/status.txt
du -sh gpurun_out >> gpurun_out/status.txt
