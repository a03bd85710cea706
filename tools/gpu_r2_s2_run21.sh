mkdir -p gpurun_out/s2
timeout 120 python tools/diag_codec3.py 1 1.0 1 > gpurun_out/s2/diag_fix.txt 2>&1; echo rc=$?
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3h_kernels.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_decode_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3h_decode.txt 2>&1; echo rc=$?
for m in 64 256; do timeout 300 python tools/profile_kernels.py --mu $m --codec3 > gpurun_out/s2/prof_c3h_mu$m.txt 2>&1; done
