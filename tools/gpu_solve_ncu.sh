#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"^k_bwd_mma4$" --launch-skip 3 --launch-count 1 -o gpurun_out/sol_bwdm_l11 -f python tools/solve_check.py 1 > gpurun_out/sol_ncu1.log 2>&1; echo "ncu1 rc=$?"
