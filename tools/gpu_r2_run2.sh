set -x
mkdir -p gpurun_out/r2
export MLT_PARITY_OUT=gpurun_out/r2/headline_parity.json
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/r2/t_attn.txt 2>&1; echo rc=$?
for g in 2 3 4; do timeout 300 python tools/profile_kernels.py --mu 64 --codec --dec-groups $g > gpurun_out/r2/prof_codec_g$g.txt 2>&1; echo rc=$?; done
timeout 300 python tools/profile_kernels.py --mu 64 > gpurun_out/r2/prof_raw.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_tp_gpu.py -x -q -s > gpurun_out/r2/t_tp.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_headline_parity_gpu.py -x -q -s > gpurun_out/r2/t_headline.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_headline_parity_gpu.py::test_headline_config_parity > gpurun_out/r2/t_gpu.txt 2>&1; echo rc=$?
