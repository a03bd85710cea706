set -x
mkdir -p gpurun_out/s2
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3_kernels.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 > gpurun_out/s2/prof_codec3_mu64.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --down-splits 1 > gpurun_out/s2/prof_codec3_mu64_ds1.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec3 > gpurun_out/s2/prof_codec3_mu256.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec > gpurun_out/s2/prof_codec_mu256.txt 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3_decode.txt 2>&1; echo rc=$?
