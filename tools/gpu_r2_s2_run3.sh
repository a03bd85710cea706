set -x
mkdir -p gpurun_out/s2
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3b_kernels.txt 2>&1; echo rc=$?
for m in 64 256; do timeout 300 python tools/profile_kernels.py --mu $m --codec3 > gpurun_out/s2/prof_codec3b_mu$m.txt 2>&1; done
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --down-splits 1 > gpurun_out/s2/prof_codec3b_mu64_ds1.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --down-splits 2 > gpurun_out/s2/prof_codec3b_mu64_ds2.txt 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3b_decode.txt 2>&1; echo rc=$?
