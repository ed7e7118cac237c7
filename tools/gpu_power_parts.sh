# energy per component: the power probe over cost-probe builds (uniform inputs)
V=paper_2310_03294_b200/variants
timeout 300 python tools/power_probe.py 4 2>&1 | grep uniform | sed 's/^/product   /'
DISTATTN_B200_LIB=$V/lib_b_noreduce.so timeout 300 python tools/power_probe.py 4 2>&1 | grep -E "^backward +uniform" | sed 's/^/no-dQ-reduce   /'
DISTATTN_B200_LIB=$V/lib_b_mma.so timeout 300 python tools/power_probe.py 4 2>&1 | grep -E "^backward +uniform" | sed 's/^/bwd-MMA-only   /'
DISTATTN_B200_LIB=$V/lib_f_mma.so timeout 300 python tools/power_probe.py 4 2>&1 | grep -E "^forward +uniform" | sed 's/^/fwd-MMA-only   /'
