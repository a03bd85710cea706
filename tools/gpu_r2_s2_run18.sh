mkdir -p gpurun_out/s2
for cfg in "4 4096 14336 8 2 16 2 1 1" "4 4096 14336 8 2 16 2 1 0" "4 4096 14336 8 2 16 2 0 1" "64 4096 14336 8 2 64 2 1 1" "4 1024 3584 8 2 16 2 1 1"; do
  timeout 60 python tools/diag_codec3_raw.py $cfg 2>&1 | tail -n 1
done > gpurun_out/s2/diag_raw_bisect2.txt
