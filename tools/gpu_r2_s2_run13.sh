mkdir -p gpurun_out/s2
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_memcheck1.txt 2>&1; echo rc=$?
