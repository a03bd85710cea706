mkdir -p gpurun_out/s2
timeout 300 python tools/ktrace3.py --mu 64 > gpurun_out/s2/ktrace3_gu.txt 2>&1
timeout 300 python tools/ktrace3.py --mu 64 --down > gpurun_out/s2/ktrace3_dn.txt 2>&1
