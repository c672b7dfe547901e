#!/bin/bash
# round-2 first GPU pass: smoke, GPU tests, a short C4 bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02i_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02i_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -s --durations=20 > gpurun_out/r02i_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
timeout 1200 python bench.py --steps 2 --warmup 3 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
echo "bench rc=$?" >> gpurun_out/r02i_bench.err
