set -x
mkdir -p gpurun_out/r2
export MLT_PARITY_OUT=gpurun_out/r2/headline_parity.json
./tools/mma_probe > gpurun_out/r2/mma_probe.txt 2>&1
for m in 16 32; do timeout 300 python tools/profile_kernels.py --mu $m > gpurun_out/r2/prof_raw_mu$m.txt 2>&1; done
timeout 900 python -m pytest tests/test_tp_gpu.py tests/test_cpp_api_gpu.py -x -q -s > gpurun_out/r2/t_tp.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_headline_parity_gpu.py -x -q -s > gpurun_out/r2/t_headline.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_decode_gpu.py -q -s > gpurun_out/r2/t_decode.txt 2>&1; echo rc=$?
