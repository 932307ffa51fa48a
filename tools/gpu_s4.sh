#!/usr/bin/env bash
# Round-2 measurement set C: seg_small (one warp per small output) + heev placement rule:
# parity suite, A/B benches, per-shape profile, ncu of the configs[2] level-12 target sums,
# C++ drop-in timing with the parallel flatten, arena-cap diagnostic.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for c in cfg3 cfg5s cfg2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
done
for c in cfg3 cfg5s; do
  H2B_SMALL_MAXCH=0 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_nosmall.json 2> gpurun_out/bench_${c}_nosmall.err; echo "bench $c nosmall rc=$?" >> gpurun_out/status.txt
  H2B_SMALL_MAXCH=1000 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_allsmall.json 2> gpurun_out/bench_${c}_allsmall.err; echo "bench $c allsmall rc=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/shape_profile.py cfg3 40 > gpurun_out/shapes_cfg3.txt 2>&1
timeout 300 python tools/shape_profile.py cfg5s 40 > gpurun_out/shapes_cfg5s.txt 2>&1
g++ -std=c++17 -O2 -Iinclude tools/dropin_time.cpp -Lpaper_1908_05218_b200/lib -lh2mmp_b200 -Wl,-rpath,$PWD/paper_1908_05218_b200/lib -pthread -o /tmp/dropin_time &&
timeout 900 /tmp/dropin_time > gpurun_out/dropin_time_cfg2.json 2> gpurun_out/dropin_time_cfg2.err; echo "dropin_time rc=$?" >> gpurun_out/status.txt
export H2B_NVTX=1
export H2B_ARENA_GB=40
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "L12.targets:seg_gemm]" \
    -c 8 -o gpurun_out/l12_cfg3 -f python tools/one_product.py cfg3 > gpurun_out/ncu_l12_cfg3.log 2>&1
echo "ncu L12 cfg3 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh l12_cfg3 >> gpurun_out/status.txt 2>&1
unset H2B_NVTX
H2B_ARENA_GB=80 H2B_MEM_TRACE=1 timeout 600 python -X faulthandler tools/one_product.py cfg5 > gpurun_out/arena80_cfg5.out 2> gpurun_out/arena80_cfg5.err; echo "arena80 cfg5 rc=$?" >> gpurun_out/status.txt
tail -c 20000 gpurun_out/arena80_cfg5.err > gpurun_out/arena80_cfg5.err.tail; rm -f gpurun_out/arena80_cfg5.err
echo done >> gpurun_out/status.txt
du -sh gpurun_out >> gpurun_out/status.txt
