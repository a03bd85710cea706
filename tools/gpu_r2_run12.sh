set -x
mkdir -p gpurun_out/r2
for t in 8 4; do timeout 900 python bench.py --config dbrx-tp --tp-shard $t --steps 128 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_dbrx_shard$t.json 2> gpurun_out/r2/bench_dbrx_shard$t.err; echo rc=$?; done
timeout 900 python bench.py --config mixtral8x7b-resident --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_resident.json 2> gpurun_out/r2/bench_resident.err; echo rc=$?
timeout 900 python bench.py --config mixtral8x7b-resident --steps 10 --warmup 3 --no-cpu-baseline --no-pdl > gpurun_out/r2/bench_resident_nopdl.json 2> gpurun_out/r2/bench_resident_nopdl.err; echo rc=$?
