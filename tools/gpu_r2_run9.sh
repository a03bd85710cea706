set -x
mkdir -p gpurun_out/r2
export MLT_PARITY_OUT=gpurun_out/r2/headline_parity.json
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2/t_gpu_all.txt 2>&1; echo rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --roofline-csv gpurun_out/r2/roofline_default.csv > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err; echo rc=$?
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err; echo rc=$?
timeout 600 python tools/tiny_cpu_gpu.py --out gpurun_out/r2/tiny_cpu_gpu.json > /dev/null 2> gpurun_out/r2/tiny.err; echo rc=$?
