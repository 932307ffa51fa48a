#!/bin/bash
# GPU box: bench (default cfg5) + reference arm on the same config, outputs into gpurun_out/
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
free -g > gpurun_out/mem_before.txt
( while true; do free -g | awk 'NR==2{print $3}' >> gpurun_out/mem_trace.txt; sleep 5; done ) &
MT=$!
timeout 1500 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo "bench rc=$?" >> gpurun_out/status.txt
timeout 1200 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/ref_cfg5.json 2> gpurun_out/ref_cfg5.err
echo "ref rc=$?" >> gpurun_out/status.txt
kill $MT
