# Round profile: default bench line, ncu launch list of the bench command,
# full ncu captures of the top kernels (tools/profile_step.py at C4).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:^k_green_jvp$ -s 0 -c 1 -o gpurun_out/green_jvp python tools/profile_step.py > gpurun_out/ncu_gj.log 2>&1
timeout 600 $N -k regex:^k_green_vjp$ -s 0 -c 1 -o gpurun_out/green_vjp python tools/profile_step.py > gpurun_out/ncu_gv.log 2>&1
timeout 600 $N -k regex:k_gemm6 -s 64 -c 1 -o gpurun_out/gemm8_l64 python tools/profile_step.py > gpurun_out/ncu_g8.log 2>&1
