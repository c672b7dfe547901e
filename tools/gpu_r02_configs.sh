#!/bin/bash
# other configs on the final code: C2 (shifted-solve microbenchmark), C3 (Jacobian
# operator benchmark), C5 rank-0 shard of an 8-GPU run
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --config C2 --no-cpu --no-c1 > gpurun_out/r02d_c2.json 2> gpurun_out/r02d_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config C3 --no-cpu --no-c1 > gpurun_out/r02d_c3.json 2> gpurun_out/r02d_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config C5 --shard 8 --no-cpu --no-c1 > gpurun_out/r02d_c5.json 2> gpurun_out/r02d_c5.err; echo "c5 rc=$?"
tail -c 600 gpurun_out/r02d_c5.err
