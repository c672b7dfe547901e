# A/B helper over environment settings: GPU tests once (defaults), then a short
# C4 bench per setting.  usage: bash tools/gpu_ab_env.sh "A=1,B=2 A=0" [pytest-args]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${2:-} > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
i=0
for tok in $1; do
  i=$((i+1))
  env $(echo $tok | tr ',' ' ') timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/abe_$i.log 2>&1
  echo "$tok" >> gpurun_out/abe_$i.log
done
