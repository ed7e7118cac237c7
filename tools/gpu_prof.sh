# usage: TAG=r1h bash tools/gpu_prof.sh
# full ncu captures of both kernels at the bench size, DRAM traffic per launch
# inside the bench step, and the launch list of the bench command
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_${TAG:-r1h} python tools/probe.py 32 32768 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_${TAG:-r1h} python tools/probe.py 32 32768 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_ -s 6 -c 2 --csv --log-file gpurun_out/traffic_${TAG:-r1h}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG:-r1h}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
