# round 2 session 3: codec-4 re-measure of Config 3 (mu 64, both placements) and the TP shards
mkdir -p gpurun_out/s3
timeout 1500 python tools/hrm_sweep.py --budgets 16,32,64 --mus 64 --codec --out gpurun_out/s3/hrm_sweep_codec4_mu64.json > gpurun_out/s3/hrm_sweep.log 2>&1; echo sweep rc=$?
for t in 8 4 2; do timeout 900 python bench.py --config mixtral8x22b-tp --tp-shard $t --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_8x22b_shard$t.json 2> gpurun_out/s3/bench_8x22b_shard$t.err; echo 8x22b $t rc=$?; done
for t in 8 4 2; do timeout 900 python bench.py --config dbrx-tp --tp-shard $t --steps 128 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_dbrx_shard$t.json 2> gpurun_out/s3/bench_dbrx_shard$t.err; echo dbrx $t rc=$?; done
