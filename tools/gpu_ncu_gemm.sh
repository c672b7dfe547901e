mkdir -p gpurun_out
RBA_GEMM=v6c timeout 300 python tools/profile_step.py > gpurun_out/ps_v6c.log 2>&1 && \
RBA_GEMM=v6c timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm6 -s 64 -c 1 -o gpurun_out/gemm6c_l64 -f python tools/profile_step.py > gpurun_out/ncu_g6.log 2>&1
RBA_GEMM=v5 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm5 -s 64 -c 1 -o gpurun_out/gemm5_l64 -f python tools/profile_step.py > gpurun_out/ncu_g5.log 2>&1
