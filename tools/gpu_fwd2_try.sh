nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
DA_FWD_KERNEL=pair timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "fwd_diagonal_finalize" 2>&1 | tail -15
echo "rc=$?"
DA_FWD_KERNEL=pair timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "fwd or chain or peaky" 2>&1 | tail -15
timeout 120 python tools/probe.py 32 32768 2>&1 | head -1
DA_FWD_KERNEL=pair timeout 120 python tools/probe.py 32 32768 2>&1 | head -1
timeout 120 python tools/probe.py 32 32768 2>&1 | head -1
DA_FWD_KERNEL=pair timeout 120 python tools/probe.py 32 32768 2>&1 | head -1
