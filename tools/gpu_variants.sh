for v in default novec default novec; do
  if [ $v = default ]; then L=paper_2310_03294_b200/libdistattn_b200.so; else L=paper_2310_03294_b200/variants/lib_$v.so; fi
  echo "== $v"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^bwd  "
done
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_novec_trace.so timeout 120 python tools/trace_bwd.py 32768 2>&1 | tail -3
