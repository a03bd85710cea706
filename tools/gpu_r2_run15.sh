set -x
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r2/t_attn3.txt 2>&1; echo rc=$?
for m in 16 32 64 128 256; do timeout 300 python tools/profile_kernels.py --mu $m > gpurun_out/r2/prof_attn3_mu$m.txt 2>&1; done
