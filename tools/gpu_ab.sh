# A/B helper: factor parity of every GEMM variant, then short C4 benches.
# usage: bash tools/gpu_ab.sh "v5 v6c v7:v6c"   (schur[:panel] kernel choices)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_factor_structure.py -x -q -s -k dmma > gpurun_out/ab_fs.log 2>&1; echo "rc=$?" >> gpurun_out/ab_fs.log
for tok in $1; do
  g=${tok%%:*}; p=${tok#*:}; [ "$p" = "$tok" ] && p=""
  RBA_GEMM=$g RBA_GEMM_PANEL=$p timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ab_bench_${g}_${p}.log 2>&1
done
