# backward head grouping under GQA (cfg2gqa): forced 1 vs 2 kv heads per grid group
for r in 1 2; do for v in hg1 hg2; do
  DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_$v.so timeout 300 python bench.py --config cfg2gqa --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k: round(x,3) for k,x in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
