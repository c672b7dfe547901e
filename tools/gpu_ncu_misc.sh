# ncu --set full captures of the non-GEMM factorisation kernels at C4:
# TRSM and extend-add at level 11, the diagonal-block kernel at level 0.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:k_gemm3 -s 200 -c 1 -o gpurun_out/trsm_mid python tools/profile_step.py > gpurun_out/ncu_t.log 2>&1
timeout 600 $N -k regex:^k_extend_add$ -s 11 -c 1 -o gpurun_out/ea_l11 python tools/profile_step.py > gpurun_out/ncu_ea.log 2>&1
timeout 600 $N -k regex:^k_diag2$ -s 0 -c 1 -o gpurun_out/diag_l0 python tools/profile_step.py > gpurun_out/ncu_d0.log 2>&1
