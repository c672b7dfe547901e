#!/bin/bash
# TS (A operand from TMEM) Ozaki GEMM: probe, bitwise test, C4 factor A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_ts_probe tools/umma_i8_ts_probe.cu && \
  timeout 120 tools/umma_i8_ts_probe > gpurun_out/r02w_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/r02w_probe.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ozaki.py > gpurun_out/r02w_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02w_pytest.log
for v in 0 1; do
  RBA_OZ_TS=$v timeout 600 python tools/oz_check.py > gpurun_out/r02w_oz$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r02w_oz$v.log
done
