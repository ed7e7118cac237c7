set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2310_03294_b200/build.py
timeout 180 python -m pytest tests/test_gpu_kernels.py -q -k "debug" -x 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "fwd or rescale" 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "bwd and not 32k" 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "32k" 2>&1 | tail -15
timeout 300 python tools/probe.py 32 32768 2>&1 | tail -5
