set -x
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_tp_gpu.py -q -s > gpurun_out/r2/t_tp2.txt 2>&1; echo rc=$?
ncu --metrics gpu__time_duration.sum -c 1 python -c "import os, torch; print('AFF', len(os.sched_getaffinity(0)), os.cpu_count(), os.environ.get('OMP_NUM_THREADS')); torch.zeros(1, device='cuda')" > gpurun_out/r2/ncu_probe.txt 2>&1
python -c "import os; print('AFF-noncu', len(os.sched_getaffinity(0)))" >> gpurun_out/r2/ncu_probe.txt 2>&1
