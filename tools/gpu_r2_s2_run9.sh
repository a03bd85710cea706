mkdir -p gpurun_out/s2
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3e_kernels.txt 2>&1; echo rc=$?
for nc in 64 32; do
  timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --ncap-e $nc > gpurun_out/s2/prof_c3e_ncap$nc.txt 2>&1
done
timeout 300 python tools/profile_kernels.py --mu 64 --codec --ncap-e 32 > gpurun_out/s2/prof_c1e_ncap32.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec3 > gpurun_out/s2/prof_c3e_mu256.txt 2>&1
timeout 300 python tools/ktrace3.py --mu 64 > gpurun_out/s2/ktrace3e_gu.txt 2>&1
timeout 300 python tools/ktrace3.py --mu 64 --down > gpurun_out/s2/ktrace3e_dn.txt 2>&1
