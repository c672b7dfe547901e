#!/bin/bash
# round-2 profiles: (1) bench without ncu, (2) launch list of the same bench
# command (gpu__time_duration.sum, clock-control none), (3) one ncu --set full
# capture of the top kernel (k_oz_gemm) and of the DMMA GEMM, from oz_check
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 1 --warmup 3 --no-c1 --no-cpu --no-verify > gpurun_out/r02prof_bench.json 2> gpurun_out/r02prof_bench.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/r02prof_launches.csv python bench.py --steps 1 --warmup 3 --no-c1 --no-cpu --no-verify \
  > gpurun_out/r02prof_ncu.log 2>&1
echo "launches rc=$?" >> gpurun_out/r02prof_ncu.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_oz_gemm|k_gemm6" \
  --launch-skip 60 --launch-count 2 -o gpurun_out/r02prof_full python tools/oz_check.py > gpurun_out/r02prof_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r02prof_full.log
