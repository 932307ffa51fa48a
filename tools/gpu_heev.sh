#!/bin/bash
# GPU box: eigensolver tests + a few parity tests + smoke + cfg5/cfg2 bench (profile) with the engine's solver
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "truncation" > gpurun_out/t_heev.txt 2>&1
echo "heev tests rc=$?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matches_oracle or cfg1 or complex or small_tile" > gpurun_out/t_parity.txt 2>&1
echo "parity rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo "bench5 rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 2 --profile --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
echo "bench2 rc=$?" >> gpurun_out/status.txt
