set -x
mkdir -p gpurun_out/r2
timeout 600 python tools/tiny_cpu_gpu.py --out gpurun_out/r2/tiny_cpu_gpu.json > /dev/null 2> gpurun_out/r2/tiny.err; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2/ncu_bench.log 2>&1; echo rc=$?
timeout 1800 python tools/hrm_sweep.py --codec --budgets 16,32,64 --mus 16,32,64,128,256 --steps 2 --out gpurun_out/r2/hrm_sweep_codec.json > /dev/null 2> gpurun_out/r2/hrm_sweep_codec.err; echo rc=$?
for t in 8 4; do timeout 900 python bench.py --config dbrx-tp --tp-shard $t --steps 128 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_dbrx_shard$t.json 2> gpurun_out/r2/bench_dbrx_shard$t.err; echo rc=$?; done
