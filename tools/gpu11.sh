mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; tail -1 gpurun_out/bench_r1.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1.json 2>&1; tail -1 gpurun_out/bench_ref_r1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_r1b python tools/probe.py 32 16384 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_r1b python tools/probe.py 32 16384 > /dev/null 2>&1
ls gpurun_out
