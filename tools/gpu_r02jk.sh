#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
bash tools/gpu_r02k.sh
date +%s > gpurun_out/r02j_t0
bash tools/gpu_r02j.sh
date +%s > gpurun_out/r02j_t1
