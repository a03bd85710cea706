mkdir -p gpurun_out/s2
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s2/gputests_c3.txt 2>&1; echo rc=$?
for ds in 1 2 4 8; do timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --down-splits $ds > gpurun_out/s2/prof_c3_ds$ds.txt 2>&1; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s2/bench_default.json 2> gpurun_out/s2/bench_default.err; echo rc=$?
