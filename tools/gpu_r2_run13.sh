set -x
mkdir -p gpurun_out/r2
for s in 2 4; do timeout 900 python bench.py --config mixtral8x7b-resident --steps 10 --warmup 3 --no-cpu-baseline --down-splits $s > gpurun_out/r2/bench_resident_ds$s.json 2> gpurun_out/r2/bench_resident_ds$s.err; echo rc=$?; done
for s in 2 4; do timeout 300 python tools/profile_kernels.py --mu 64 --down-splits $s > gpurun_out/r2/prof_raw_ds$s.txt 2>&1; done
timeout 300 python tools/profile_kernels.py --mu 256 > gpurun_out/r2/prof_raw_mu256.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --down-splits 4 > gpurun_out/r2/prof_raw_mu256_ds4.txt 2>&1
timeout 600 python bench.py --config tiny --steps 31 --warmup 3 > gpurun_out/r2/bench_tiny.json 2> gpurun_out/r2/bench_tiny.err; echo rc=$?
timeout 600 python bench.py --config tiny --impl reference --steps 31 --warmup 3 > gpurun_out/r2/bench_tiny_ref.json 2> gpurun_out/r2/bench_tiny_ref.err; echo rc=$?
