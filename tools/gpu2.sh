set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -3
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -c 2 -o gpurun_out/prof_r1 python tools/probe.py 32 16384 > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
