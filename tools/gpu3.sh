mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -c 1 -o gpurun_out/prof_bwd_r1 python tools/probe.py 32 16384 > gpurun_out/ncu_bwd.log 2>&1
tail -3 gpurun_out/ncu_bwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_fwd_r1 python tools/probe.py 32 16384 > gpurun_out/ncu_fwd.log 2>&1
tail -3 gpurun_out/ncu_fwd.log
