#!/usr/bin/env bash
# Round-2 measurement set F: A/B of the accumulate-tile L2 prefetch, parity suite on the final
# kernels, default bench line, reference arm twice (constructor, then the disk cache).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in cfg5s cfg2 cfg3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/status.txt
  H2B_NO_CPREFETCH=1 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_${c}_nocpf.json 2> gpurun_out/bench_${c}_nocpf.err; echo "bench $c nocpf rc=$?" >> gpurun_out/status.txt
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 1500 python bench.py --steps 5 --warmup 3 --profile > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench cfg5 rc=$?" >> gpurun_out/status.txt
H2B_NO_CPREFETCH=1 timeout 1500 python bench.py --steps 5 --warmup 3 --profile --no-cpu > gpurun_out/bench_cfg5_nocpf.json 2> gpurun_out/bench_cfg5_nocpf.err; echo "bench cfg5 nocpf rc=$?" >> gpurun_out/status.txt
( time timeout 1800 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err ) 2> gpurun_out/bench_reference.time; echo "bench reference rc=$?" >> gpurun_out/status.txt
( time timeout 1800 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_cached.json 2> gpurun_out/bench_reference_cached.err ) 2> gpurun_out/bench_reference_cached.time; echo "bench reference cached rc=$?" >> gpurun_out/status.txt
ls -la /tmp/h2b_bench_cache >> gpurun_out/status.txt 2>&1
echo done >> gpurun_out/status.txt
