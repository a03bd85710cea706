mkdir -p gpurun_out/s2
MLT_SYNC_EACH=1 timeout 120 python tools/diag_codec3.py 1 1.0 1 > gpurun_out/s2/diag_printf.txt 2>&1; echo rc=$?
MLT_NO_STREAM_K=1 MLT_SYNC_EACH=1 timeout 120 python tools/diag_codec3.py 1 1.0 1 > gpurun_out/s2/diag_printf_nosk.txt 2>&1; echo rc=$?
