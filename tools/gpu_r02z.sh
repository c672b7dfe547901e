#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" RBA_OZ_STAGES=4 timeout 600 python tools/oz_check.py > gpurun_out/r02z_oz_$tag.log 2>&1; echo "== $tag: $@"; grep -h "oz_prof\|factor 16\|classes" gpurun_out/r02z_oz_$tag.log; }
run a RBA_OZ_TRAIL=1 RBA_PANEL=4 RBA_OZ_MINROWS=256 RBA_OZ_MINK=128
run g RBA_OZ_TRAIL=1 RBA_PANEL=4 RBA_OZ_MINROWS=512 RBA_OZ_MINK=256
