# sustained A/B: working-tree library vs the committed build (variants/lib_base.so)
D=paper_2310_03294_b200/libdistattn_b200.so
B=paper_2310_03294_b200/variants/lib_base.so
for r in 1 2 3; do for L in $D $B; do timeout 120 python tools/ab_step.py $L 4; done; done
