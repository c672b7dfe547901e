#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_oz|k_gemm6|k_extend|k_diag2|k_gemm3|k_zbwd|k_fwd|k_bwd|k_green" --launch-skip 1500 --launch-count 1500 --csv --log-file gpurun_out/r02o_launches.csv python tools/oz_check.py > gpurun_out/r02o.log 2>&1
echo "rc=$?" >> gpurun_out/r02o.log
