set -x
mkdir -p gpurun_out/r2
timeout 600 ncu --set full --clock-control none -k regex:gemm_codec -c 4 -o gpurun_out/r2/ncu_codec2 python tools/profile_kernels.py --mu 64 --codec2 --once > gpurun_out/r2/ncu_codec2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc -c 12 -o gpurun_out/r2/ncu_codec1 python tools/profile_kernels.py --mu 64 --codec --once > gpurun_out/r2/ncu_codec1.log 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "codec" > gpurun_out/r2/t_codec2_kern.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_prefill_gpu.py tests/test_codec_ingest_gpu.py -q -x -s -k "codec" > gpurun_out/r2/t_codec2_dec.txt 2>&1; echo rc=$?
