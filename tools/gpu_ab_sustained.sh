for v in ${VARIANTS:-default nodq default nodq}; do
  if [ $v = default ]; then L=paper_2310_03294_b200/libdistattn_b200.so; else L=paper_2310_03294_b200/variants/lib_$v.so; fi
  echo "== $v"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^(fwd|bwd)  "
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader
done
