#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/r02j_host.txt; free -g >> gpurun_out/r02j_host.txt
timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02j_ref.json 2> gpurun_out/r02j_ref.err
echo "ref rc=$?" >> gpurun_out/r02j_ref.err
