set -x
mkdir -p gpurun_out/r2
nproc; free -g | head -2
export MLT_PARITY_OUT=gpurun_out/r2/headline_parity.json
timeout 900 python -m pytest tests/test_headline_parity_gpu.py -x -q -s > gpurun_out/r2/t_headline.txt 2>&1; echo rc=$?
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2/t_gpu.txt 2>&1; echo rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --roofline-csv gpurun_out/r2/roofline.csv > gpurun_out/r2/b1.json 2> gpurun_out/r2/b1.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2/r1.json 2> gpurun_out/r2/r1.err; echo rc=$?
