#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python bench.py --config C5 --shard 8 --warmup 1 > gpurun_out/r02q_c5.json 2> gpurun_out/r02q_c5.err
echo "rc=$?" >> gpurun_out/r02q_c5.err
