mkdir -p gpurun_out/s2
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_blk.txt 2>&1; echo rc=$?
MLT_NO_STREAM_K=1 timeout 300 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_nosk.txt 2>&1; echo rc=$?
timeout 300 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_again.txt 2>&1; echo rc=$?
