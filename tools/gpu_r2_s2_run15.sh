mkdir -p gpurun_out/s2
MLT_SYNC_EACH=1 timeout 300 python tools/diag_codec3.py 1 > gpurun_out/s2/diag_sync.txt 2>&1; echo rc=$?
