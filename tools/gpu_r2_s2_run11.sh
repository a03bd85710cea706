mkdir -p gpurun_out/s2
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3g_kernels.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 > gpurun_out/s2/prof_c3g_mu64.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec3 > gpurun_out/s2/prof_c3g_mu256.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 32 --codec3 > gpurun_out/s2/prof_c3g_mu32.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 128 --codec3 > gpurun_out/s2/prof_c3g_mu128.txt 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3g_decode.txt 2>&1; echo rc=$?
