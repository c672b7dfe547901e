#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eight_rhs or solves_vs_splu" -s > gpurun_out/r02r_pytest.log 2>&1
RBA_BWD_GEMM=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solves_vs_splu or c1_full or forward_jvp" -s >> gpurun_out/r02r_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02r_pytest.log
RBA_BWD_GEMM=1 timeout 600 python tools/oz_check.py 2>&1 | tail -3 > gpurun_out/r02r_oz.log
timeout 1500 python bench.py --config C5 --shard 8 --warmup 1 > gpurun_out/r02r_c5.json 2> gpurun_out/r02r_c5.err
