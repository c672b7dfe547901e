#!/bin/bash
# wide-N Ozaki MMAs: bitwise test, C4 factor A/B (wide / narrow), ncu of the wide kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ozaki.py > gpurun_out/r02y_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02y_pytest.log
RBA_OZ_WIDE=1 timeout 600 python tools/oz_check.py > gpurun_out/r02y_oz_wide.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_oz_wide.log
RBA_OZ_WIDE=0 timeout 600 python tools/oz_check.py > gpurun_out/r02y_oz_narrow.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_oz_narrow.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_oz_gemm" \
  --launch-skip 16 --launch-count 1 -o gpurun_out/r02y_ozwide -f python tools/oz_check.py > gpurun_out/r02y_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02y_ncu.log
for f in gpurun_out/r02y_*.log; do echo "== $f"; tail -n 4 $f; done
