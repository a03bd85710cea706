# round 2 session 3: codec-4 capacity per weight kind — tests, headline bench, DBRX shards (fell back to codec 3 before)
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_decode_gpu.py tests/test_codec_ingest_gpu.py -m gpu -q -k "codec" > gpurun_out/s3/tests_cap.txt 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3/tests_cap.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3/bench_default3.json 2> gpurun_out/s3/bench_default3.err; echo bench rc=$?
for t in 8 2 4; do timeout 900 python bench.py --config dbrx-tp --tp-shard $t --steps 128 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_dbrx_cap_shard$t.json 2> gpurun_out/s3/bench_dbrx_cap_shard$t.err; echo dbrx $t rc=$?; done
