# e2e pipeline: heads per group (copy/compute granularity) A/B
D=paper_2310_03294_b200/libdistattn_b200.so
for r in 1 2; do for g in 2 4 8 1; do echo "hpg=$g"; timeout 120 python tools/ab_e2e.py $D 4 $g; done; done
