timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py -q -x 2>&1 | tail -1
for i in 1 2; do timeout 120 python tools/probe.py 32 32768 | tail -3; done
for i in 1 2; do DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_headminor.so timeout 120 python tools/probe.py 32 32768 | tail -3; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_ -s 6 -c 2 --csv --log-file gpurun_out/traffic_r1b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cut -d, -f5,13,15 gpurun_out/traffic_r1b.csv | tail -6
