set -x
mkdir -p gpurun_out/r2
for g in 1 2; do timeout 300 python tools/profile_kernels.py --mu 64 --codec --dec-groups $g > gpurun_out/r2/prof_codec_dg$g.txt 2>&1; echo rc=$?; done
timeout 300 python tools/ktrace_gemm.py --down --dec-groups 1 > gpurun_out/r2/ktrace_down_dg1.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 256 --codec --dec-groups 1 > gpurun_out/r2/prof_codec_dg1_mu256.txt 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "codec" > gpurun_out/r2/t_codec_kern.txt 2>&1; echo rc=$?
