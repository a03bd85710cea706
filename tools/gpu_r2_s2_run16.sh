mkdir -p gpurun_out/s2
for cfg in "4 4096 14336 8 2 16 2" "4 4096 1024 8 2 16 2" "4 1024 14336 8 2 16 2" "4 2048 2048 8 2 16 2" "4 4096 14336 8 2 16 1" "64 4096 2048 8 2 64 2" "4 3072 1024 8 2 16 2" "4 2048 1024 8 2 16 1"; do
  timeout 120 python tools/diag_codec3_raw.py $cfg 2>&1 | tail -n 1
done > gpurun_out/s2/diag_raw_bisect.txt
