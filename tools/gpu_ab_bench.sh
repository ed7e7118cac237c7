# A/B of library variants inside the sustained bench step (kernel_ms per kernel):
# VARIANTS="default g1 default g1" bash tools/gpu_ab_bench.sh
for v in ${VARIANTS:-default g1 default g1}; do
  if [ $v = default ]; then L=paper_2310_03294_b200/libdistattn_b200.so; else L=paper_2310_03294_b200/variants/lib_$v.so; fi
  printf "%-10s " $v
  DISTATTN_B200_LIB=$L timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(x, 3) for k, x in d['kernel_ms'].items()}, 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
