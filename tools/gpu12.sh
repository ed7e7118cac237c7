timeout 400 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_ -s 6 -c 2 --csv --log-file gpurun_out/traffic_r1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/traffic_r1.csv | tail -8
