#!/bin/bash
# re-entry check: TS probe, Ozaki tests, C4 factor A/B (SS / TS / cluster pair)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_ts_probe tools/umma_i8_ts_probe.cu && \
  timeout 120 tools/umma_i8_ts_probe > gpurun_out/r02x_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/r02x_probe.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ozaki.py > gpurun_out/r02x_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02x_pytest.log
RBA_OZAKI=1 timeout 600 python tools/oz_check.py > gpurun_out/r02x_oz_ss.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_oz_ss.log
RBA_OZAKI=1 RBA_OZ_TS=1 timeout 600 python tools/oz_check.py > gpurun_out/r02x_oz_ts.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_oz_ts.log
RBA_OZAKI=1 RBA_OZ_2CTA=1 timeout 600 python tools/oz_check.py > gpurun_out/r02x_oz_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_oz_pair.log
tail -3 gpurun_out/r02x_*.log
