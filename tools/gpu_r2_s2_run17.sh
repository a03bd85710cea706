mkdir -p gpurun_out/s2
for cfg in "1 0.10 2" "1 1.0 2" "1 0.10 1" "1 0.5 2" "1 0.10 2 4096 2048" "1 0.10 2 2048 14336" "1 0.10 2 1024 14336"; do
  echo "cfg $cfg: $(MLT_SYNC_EACH=1 timeout 120 python tools/diag_codec3.py $cfg 2>&1 | tail -n 1)"
done > gpurun_out/s2/diag_rt_bisect.txt
