# Round profile: default bench line, ncu launch list of the bench command,
# full ncu capture of the dominant kernel (level-13 Schur GEMM launch).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:k_gemm6 -s 64 -c 1 -o gpurun_out/gemm8c_l64 python tools/profile_step.py > gpurun_out/ncu_g8c.log 2>&1
