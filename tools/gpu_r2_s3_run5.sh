# round 2 session 3: half-row record bytes — tests, microbench, headline bench, DBRX tp8
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_decode_gpu.py -m gpu -q -k "codec" > gpurun_out/s3/tests_half.txt 2>&1; echo tests rc=$?; tail -1 gpurun_out/s3/tests_half.txt
for mu in 64 256; do timeout 300 python tools/profile_kernels.py --mu $mu --only expert --codec4 > gpurun_out/s3/prof_mu${mu}--codec4-half.txt 2>&1; done
grep -h "^expert" gpurun_out/s3/prof_mu64--codec4-half.txt gpurun_out/s3/prof_mu256--codec4-half.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3/bench_default4.json 2> gpurun_out/s3/bench_default4.err; echo bench rc=$?
timeout 900 python bench.py --config dbrx-tp --tp-shard 8 --steps 128 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_dbrx_half_shard8.json 2> gpurun_out/s3/bench_dbrx_half_shard8.err; echo dbrx rc=$?
