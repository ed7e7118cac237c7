# deterministic-dQ backward: working tree vs committed build (variants/lib_base.so)
for r in 1 2; do for L in paper_2310_03294_b200/libdistattn_b200.so paper_2310_03294_b200/variants/lib_base.so; do
  echo "== $L"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^bwd"
done; done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_scale.py -q -m gpu -k "determin" 2>&1 | tail -2
