#!/bin/bash
# Measures the FP64 roofline denominators on a B200 (run under gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peaks tools/fp64_peaks.cu
/tmp/fp64_peaks | tee gpurun_out/fp64_peaks.txt
python - <<'PY' | tee -a gpurun_out/fp64_peaks.txt
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM {n}^3: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
PY
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv | tee -a gpurun_out/fp64_peaks.txt
