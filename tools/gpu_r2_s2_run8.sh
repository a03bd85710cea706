mkdir -p gpurun_out/s2
for nc in 64 32 16; do
  timeout 300 python tools/profile_kernels.py --mu 64 --codec --ncap-e $nc > gpurun_out/s2/prof_c1_ncap$nc.txt 2>&1
  timeout 300 python tools/profile_kernels.py --mu 64 --codec3 --ncap-e $nc > gpurun_out/s2/prof_c3_ncap$nc.txt 2>&1
done
timeout 300 python tools/profile_kernels.py --mu 64 --ncap-e 32 > gpurun_out/s2/prof_c0_ncap32.txt 2>&1
timeout 300 python tools/ktrace_gemm.py --mu 64 > gpurun_out/s2/ktrace1_gu.txt 2>&1
timeout 300 python tools/ktrace_gemm.py --mu 64 --down > gpurun_out/s2/ktrace1_dn.txt 2>&1
