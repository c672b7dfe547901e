# Round profile: ncu launch list of the bench command and a full capture of
# the level-13 Schur GEMM launch (tools/profile_step.py at C4).
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:k_gemm6 -s 64 -c 1 -o gpurun_out/gemm8c_l64 python tools/profile_step.py > gpurun_out/ncu_g8c.log 2>&1
