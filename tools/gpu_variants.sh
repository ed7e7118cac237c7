timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^bwd"; done
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_trace.so timeout 120 python tools/trace_bwd.py 32768 2>&1 | tail -4
