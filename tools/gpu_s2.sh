#!/usr/bin/env bash
# Round-2 measurement set B1: constructor on the own kernel (tests + smoke), C++ drop-in timing,
# ncu --set full of the dominant configs[4] kernel (arena capped so ncu's replay copy fits).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ref_golden.py -x -q -m gpu -k "constructor or construction or bench_constructions or golden" > gpurun_out/t_constructor.txt 2>&1; echo "constructor tests rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg5s.json 2> gpurun_out/bench_cfg5s.err; echo "bench cfg5s rc=$?" >> gpurun_out/status.txt
g++ -std=c++17 -O2 -Iinclude tools/dropin_time.cpp -Lpaper_1908_05218_b200/lib -lh2mmp_b200 -Wl,-rpath,$PWD/paper_1908_05218_b200/lib -o /tmp/dropin_time &&
timeout 900 /tmp/dropin_time > gpurun_out/dropin_time_cfg2.json 2> gpurun_out/dropin_time_cfg2.err; echo "dropin_time rc=$?" >> gpurun_out/status.txt
export H2B_NVTX=1
export H2B_ARENA_GB=80
timeout 1500 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "leaf.full_targets:seg_gemm]" \
    -c 1 -o gpurun_out/top_cfg5 -f python tools/one_product.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo "ncu full cfg5 rc=$?" >> gpurun_out/status.txt
bash tools/ncu_export.sh top_cfg5 >> gpurun_out/status.txt 2>&1
echo done >> gpurun_out/status.txt
du -sh gpurun_out >> gpurun_out/status.txt
