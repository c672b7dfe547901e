# Round profile: default bench line, ncu launch list of the bench command,
# per-kernel DRAM bytes of tools/profile_step.py (-> profiles/dram_r01.json),
# full ncu captures of the top kernels.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_metrics.csv python tools/profile_step.py > gpurun_out/ncu_step.log 2>&1
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:^k_zbwd$ -s 14 -c 1 -o gpurun_out/zbwd_l0 python tools/profile_step.py > gpurun_out/ncu_z0.log 2>&1
timeout 600 $N -k regex:^k_zbwd$ -s 3 -c 1 -o gpurun_out/zbwd_l11 python tools/profile_step.py > gpurun_out/ncu_z11.log 2>&1
