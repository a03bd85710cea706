mkdir -p gpurun_out/s2
timeout 300 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_raw1.txt 2>&1; echo rc=$?
timeout 300 python tools/diag_codec3.py 0 > gpurun_out/s2/diag_raw0.txt 2>&1; echo rc=$?
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/diag_codec3.py 0 > gpurun_out/s2/diag_memcheck.txt 2>&1; echo rc=$?
