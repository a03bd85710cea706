set -x
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "codec" > gpurun_out/r2/t_codec2_kern.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec2 > gpurun_out/r2/prof_codec2.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 32 --codec2 > gpurun_out/r2/prof_codec2_mu32.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_prefill_gpu.py -q -x -k "codec" > gpurun_out/r2/t_codec2_dec.txt 2>&1; echo rc=$?
