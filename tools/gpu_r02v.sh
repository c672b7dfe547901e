#!/bin/bash
# round-2 re-entry: GPU tests + smoke + default bench line + launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu tests > gpurun_out/r02v_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02v_smoke.log
timeout 1500 python bench.py > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err
echo "bench rc=$?" >> gpurun_out/r02v_bench.err
