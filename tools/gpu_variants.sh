timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py -q -x 2>&1 | tail -2
for v in default pair default pair; do
  if [ $v = default ]; then L=paper_2310_03294_b200/libdistattn_b200.so; else L=paper_2310_03294_b200/variants/lib_$v.so; fi
  echo "== $v"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^fwd "
done
