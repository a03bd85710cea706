# round 2 session 3: bench with the final codec-4 engine + its ncu launch list
mkdir -p gpurun_out/s3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3/bench_default2.json 2> gpurun_out/s3/bench_default2.err; echo bench rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --only expert --codec4 > gpurun_out/s3/prof_mu64--codec4-g4.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --only expert --codec4 > gpurun_out/s3/prof_mu256--codec4-g4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 2 -o gpurun_out/s3/codec4g4_mu64 -f python tools/profile_kernels.py --mu 64 --codec4 --once --only "expert_ffn" > gpurun_out/s3/ncu_codec4g4.log 2>&1; echo ncu rc=$?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s3/ncu_bench.log 2>&1; echo launches rc=$?
