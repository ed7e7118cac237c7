timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "fwd|bwd"
