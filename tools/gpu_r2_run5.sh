set -x
mkdir -p gpurun_out/r2
timeout 300 python tools/ktrace_gemm.py --down > gpurun_out/r2/ktrace_down.txt 2>&1
timeout 300 python tools/ktrace_gemm.py > gpurun_out/r2/ktrace_gateup.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 256 --codec > gpurun_out/r2/prof_codec_kps2_mu256b.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 16 > gpurun_out/r2/prof_raw_mu16b.txt 2>&1
