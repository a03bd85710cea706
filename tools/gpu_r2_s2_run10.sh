mkdir -p gpurun_out/s2
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3f_kernels.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 > gpurun_out/s2/prof_c3f_mu64.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --ncap-e 32 > gpurun_out/s2/prof_c3f_mu64_n32.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec3 > gpurun_out/s2/prof_c3f_mu256.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 64 --codec > gpurun_out/s2/prof_c1f_mu64.txt 2>&1
timeout 300 python tools/ktrace3.py --mu 64 > gpurun_out/s2/ktrace3f_gu.txt 2>&1
