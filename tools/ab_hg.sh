# backward grid head-grouping A/B on the causal 32K and the Full 64K x 64K chunk pair (cfg4 per GPU)
V=paper_2310_03294_b200/variants
for r in 1 2; do
for L in paper_2310_03294_b200/libdistattn_b200.so $V/lib_hg1.so $V/lib_hg4.so; do
  echo "== $L"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 65536 32 full 2>&1 | grep -E "^(fwd|bwd)  "
  DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^bwd  "
done; done
