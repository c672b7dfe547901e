#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eight_rhs" -s > gpurun_out/r02s_pytest.log 2>&1
RBA_FWD_GEMM=1 RBA_BWD_GEMM=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factor_structure.py -q -x -s -k "solves_vs_splu or receiver_green or fused" >> gpurun_out/r02s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02s_pytest.log
timeout 1500 python bench.py --config C5 --shard 8 --warmup 1 > gpurun_out/r02s_c5.json 2> gpurun_out/r02s_c5.err
