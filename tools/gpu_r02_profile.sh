#!/bin/bash
# round-2 profiles: (1) bench without ncu, (2) launch list of the same bench
# command (gpu__time_duration.sum, clock-control none), (3) one ncu --set full
# capture of the top kernel (k_oz_gemm, a level-11 launch of 6 poles) and of the
# DMMA GEMM, from tools/oz_check.py
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 1 --warmup 3 --no-c1 --no-cpu --no-verify > gpurun_out/r02prof_bench.json 2> gpurun_out/r02prof_bench.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file gpurun_out/r02prof_launches.csv python bench.py --steps 1 --warmup 3 --no-c1 --no-cpu --no-verify \
  > gpurun_out/r02prof_ncu.log 2>&1
echo "launches rc=$?" >> gpurun_out/r02prof_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"^k_oz_gemm$" \
  --launch-skip 6 --launch-count 1 -o gpurun_out/r02prof_oz -f python tools/oz_check.py > gpurun_out/r02prof_full1.log 2>&1
echo "full1 rc=$?" >> gpurun_out/r02prof_full1.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"^k_gemm6$" \
  --launch-skip 300 --launch-count 1 -o gpurun_out/r02prof_gemm6 -f python tools/oz_check.py > gpurun_out/r02prof_full2.log 2>&1
echo "full2 rc=$?" >> gpurun_out/r02prof_full2.log
