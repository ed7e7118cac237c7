# where the e2e gap goes: device step (ab_step) vs the host pipeline with and without its copies
L=paper_2310_03294_b200/libdistattn_b200.so
for r in 1 2; do
  timeout 120 python tools/ab_step.py $L 6 2>&1 | tail -1 | sed 's/^/device /'
  timeout 120 python tools/ab_e2e.py $L 6 2 2>&1 | tail -1 | sed 's/^/e2e /'
  timeout 120 python tools/ab_e2e.py paper_2310_03294_b200/variants/lib_nocopy.so 6 2 2>&1 | tail -1 | sed 's/^/e2e-nocopy /'

done
