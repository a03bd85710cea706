set -x
mkdir -p gpurun_out/r2
timeout 300 python tools/profile_kernels.py --mu 64 --codec2 > gpurun_out/r2/prof_codec2b.txt 2>&1; echo rc=$?
timeout 300 python tools/profile_kernels.py --mu 64 --codec > gpurun_out/r2/prof_codec1b.txt 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "codec" > gpurun_out/r2/t_codec2_kern.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_codec_ingest_gpu.py -q -x -s > gpurun_out/r2/t_ingest.txt 2>&1; echo rc=$?
