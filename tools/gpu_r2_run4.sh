set -x
mkdir -p gpurun_out/r2
for g in 2 4; do timeout 300 python tools/profile_kernels.py --mu 64 --codec --dec-groups $g > gpurun_out/r2/prof_codec_kps2_g$g.txt 2>&1; done
timeout 300 python tools/profile_kernels.py --mu 256 --codec > gpurun_out/r2/prof_codec_kps2_mu256.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_decode_gpu.py -q -x -k "codec or gemm or expert" > gpurun_out/r2/t_codec.txt 2>&1; echo rc=$?
