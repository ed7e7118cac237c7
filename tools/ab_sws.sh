# forward S = Q K^T for both query tiles with the K operand read once (tcgen05.mma.ws B collector)
D=paper_2310_03294_b200/libdistattn_b200.so
V=paper_2310_03294_b200/variants/lib_sws.so
for r in 1 2 3; do for L in $D $V; do timeout 120 python tools/ab_step.py $L 4; done; done
DISTATTN_B200_LIB=$V timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_scale.py -q -m gpu -k "fwd or cfg2_32k_all or gqa_4to1" 2>&1 | tail -2
