set -x
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/gputests.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec > gpurun_out/s2/prof_codec_mu64.txt 2>&1
timeout 300 python tools/profile_kernels.py --mu 64 > gpurun_out/s2/prof_raw_mu64.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 2 -o gpurun_out/s2/codec_mu64 -f python tools/profile_kernels.py --mu 64 --codec --once > gpurun_out/s2/ncu_codec.log 2>&1; echo rc=$?
