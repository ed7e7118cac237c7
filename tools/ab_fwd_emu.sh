D=paper_2310_03294_b200/libdistattn_b200.so
V=paper_2310_03294_b200/variants
for r in 1 2; do
for L in $D $V/lib_emu8.so $V/lib_emu4.so $V/lib_emu3.so; do
  timeout 120 python tools/ab_step.py $L 4
done
done
