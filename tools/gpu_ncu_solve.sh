# ncu --set full captures of the top kernels at C4 (tools/profile_step.py):
# GEMM (level-13 Schur launch), big-front solves at level 11, small-front solves at level 0.
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py > gpurun_out/ps.log 2>&1 || exit 1
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:k_gemm6 -s 64 -c 1 -o gpurun_out/gemm8_l64 python tools/profile_step.py > gpurun_out/ncu_a.log 2>&1
timeout 600 $N -k regex:^k_bwd$ -s 3 -c 1 -o gpurun_out/bwd_l11 python tools/profile_step.py > gpurun_out/ncu_b.log 2>&1
timeout 600 $N -k regex:^k_fwd$ -s 4 -c 1 -o gpurun_out/fwd_l11 python tools/profile_step.py > gpurun_out/ncu_c.log 2>&1
timeout 600 $N -k regex:^k_bwd_small$ -s 6 -c 1 -o gpurun_out/bwds_l0 python tools/profile_step.py > gpurun_out/ncu_d.log 2>&1
timeout 600 $N -k regex:^k_fwd_small$ -s 0 -c 1 -o gpurun_out/fwds_l0 python tools/profile_step.py > gpurun_out/ncu_e.log 2>&1
