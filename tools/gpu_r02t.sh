#!/bin/bash
# TRSM triangular skip + cluster-pair Ozaki GEMM: tests, then C4 factor timings A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_factor_structure.py tests/test_gpu_ozaki.py > gpurun_out/r02t_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02t_pytest.log
for v in 0 1; do
  RBA_OZ_2CTA=$v timeout 600 python tools/oz_check.py > gpurun_out/r02t_oz$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r02t_oz$v.log
done
