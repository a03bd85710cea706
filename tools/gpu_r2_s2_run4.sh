set -x
mkdir -p gpurun_out/s2
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "codec" > gpurun_out/s2/t_codec3c_kernels.txt 2>&1; echo rc=$?
for m in 64 256; do timeout 300 python tools/profile_kernels.py --mu $m --codec3 > gpurun_out/s2/prof_codec3c_mu$m.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 2 -o gpurun_out/s2/codec3c_mu64 -f python tools/profile_kernels.py --mu 64 --codec3 --once > gpurun_out/s2/ncu_codec3c.log 2>&1; echo rc=$?
