set -x
nproc; lscpu | head -20; free -g; df -h /tmp | tail -1; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import os; print(len(os.sched_getaffinity(0)))"
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --profile > gpurun_out/probe_cfg5.json 2> gpurun_out/probe_cfg5.err
tail -3 gpurun_out/probe_cfg5.err
