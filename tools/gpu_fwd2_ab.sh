# sustained A/B of the CTA-pair forward (DA_FWD_KERNEL=pair) against the single-CTA kernel
L=paper_2310_03294_b200/libdistattn_b200.so
V=paper_2310_03294_b200/variants
probe() { echo "== $1"; timeout 120 python tools/probe.py 32 32768 2>&1 | grep -E "^fwd"; }
DISTATTN_B200_LIB=$V/lib_s_mma.so probe "single mma-only"
DISTATTN_B200_LIB=$V/lib_p_mma.so DA_FWD_KERNEL=pair probe "pair mma-only"
for r in 1 2; do
  timeout 120 python tools/ab_step.py $L 6 2>&1 | tail -1 | sed 's/^/single /'
  DA_FWD_KERNEL=pair timeout 120 python tools/ab_step.py $L 6 2>&1 | tail -1 | sed 's/^/pair /'
  for v in p_emu8 p_emu4 p_emu3; do
    DA_FWD_KERNEL=pair timeout 120 python tools/ab_step.py $V/lib_$v.so 6 2>&1 | tail -1 | sed 's/^/pair /'
  done
done
