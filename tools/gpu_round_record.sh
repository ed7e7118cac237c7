nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2y_gputest.log 2>&1; tail -3 gpurun_out/r2y_gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -1 gpurun_out/r2y_smoke.log
timeout 600 python bench.py > gpurun_out/r2y_bench_n1.json 2> gpurun_out/r2y_bench_n1.err; tail -c 600 gpurun_out/r2y_bench_n1.json
timeout 600 python bench.py --config cfg2gqa --no-cpu-baseline > gpurun_out/r2y_bench_gqa.json 2>&1; tail -c 300 gpurun_out/r2y_bench_gqa.json
timeout 600 python bench.py --impl reference > gpurun_out/r2y_bench_ref.json 2>&1; tail -c 300 gpurun_out/r2y_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2y.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches_r2y.csv
