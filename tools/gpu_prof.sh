# timeline traces + full ncu captures of both kernels at the bench size
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_trace.so timeout 120 python tools/trace_fwd.py 32768 2>&1 | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_r1c python tools/probe.py 32 32768 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_r1c python tools/probe.py 32 32768 > /dev/null 2>&1
ls -la gpurun_out
