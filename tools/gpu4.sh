for v in emu0 emu8 emu4 emu3 emu2; do
  echo "== $v"
  DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "fwd" 2>&1 | tail -1
  DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_$v.so timeout 300 python tools/probe.py 32 32768 2>&1 | head -1
  DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_$v.so timeout 300 python tools/probe.py 32 32768 2>&1 | head -1
done
