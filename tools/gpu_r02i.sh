#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s --durations=15 > gpurun_out/r02p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02p_pytest.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
echo "bench rc=$?" >> gpurun_out/r02p_bench.err
