# A/B of the e2e pipeline: current library vs the previous build (variants/lib_e2eold.so)
D=paper_2310_03294_b200/libdistattn_b200.so
V=paper_2310_03294_b200/variants
for r in 1 2; do
  for L in $D $V/lib_e2eold.so; do timeout 120 python tools/ab_e2e.py $L 5; done
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "host_pipeline" 2>&1 | tail -2
