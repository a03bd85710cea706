# round 2 session 3: codec 4 evidence (engines microbench, ncu capture, bench, launch list)
mkdir -p gpurun_out/s3
for mu in 64 256; do
  for v in "" "--codec3" "--codec4"; do timeout 300 python tools/profile_kernels.py --mu $mu --only expert $v > gpurun_out/s3/prof_mu${mu}${v}.txt 2>&1; done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 2 -o gpurun_out/s3/codec4_mu64 -f python tools/profile_kernels.py --mu 64 --codec4 --once --only "expert_ffn" > gpurun_out/s3/ncu_codec4.log 2>&1; echo ncu rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3/bench_default.json 2> gpurun_out/s3/bench_default.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s3/ncu_bench.log 2>&1; echo launches rc=$?
