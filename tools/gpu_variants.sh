# A/B of library variants on one box: tools/gpu_variants.sh "default lsu default lsu" [probe args]
VARIANTS=${1:-"default lsu default lsu"}; shift
for v in $VARIANTS; do
  if [ $v = default ]; then L=paper_2310_03294_b200/libdistattn_b200.so; else L=paper_2310_03294_b200/variants/lib_$v.so; fi
  echo "== $v"; DISTATTN_B200_LIB=$L timeout 120 python tools/probe.py ${@:-32 32768} 2>&1 | grep -E "^(fwd|bwd)  "
done
