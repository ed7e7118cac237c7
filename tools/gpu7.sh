DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_dqtma.so timeout 200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py -q -x 2>&1 | tail -2
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_dqtma_trace.so timeout 120 python tools/trace_bwd.py 16384
for i in 1 2; do DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_dqtma.so timeout 120 python tools/probe.py 32 32768 | tail -2; done
for i in 1 2; do timeout 120 python tools/probe.py 32 32768 | tail -2; done
