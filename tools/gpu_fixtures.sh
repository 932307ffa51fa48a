#!/bin/bash
# GPU box: all-cores oracle fixtures for the full-size parity tests (tests/golden/full_<cfg>.npz)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out tests/golden
timeout 3000 python tools/make_fixtures.py "$@" > gpurun_out/fixtures.log 2>&1
echo "fixtures rc=$?" >> gpurun_out/status.txt
mkdir -p gpurun_out/golden; cp tests/golden/full_*.npz gpurun_out/golden/ 2>/dev/null
timeout 1500 python -m pytest tests/test_full_size_fixtures.py -q -x > gpurun_out/t_fixtures.txt 2>&1
echo "fixture tests rc=$?" >> gpurun_out/status.txt
