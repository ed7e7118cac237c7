# N>1 lines with every rank sharing one GPU (IPC transport): cfg3 at full size over 2 and 8 ranks,
# cfg5 over 8 ranks, default schedules (balanced_split forward and backward)
timeout 1200 python bench.py --gpus 2 --share-gpu --steps 2 --warmup 3 > gpurun_out/r2x_n2share_cfg3.json 2> gpurun_out/r2x_n2share_cfg3.err; tail -c 400 gpurun_out/r2x_n2share_cfg3.json
timeout 1500 python bench.py --gpus 8 --share-gpu --steps 1 --warmup 3 > gpurun_out/r2x_n8share_cfg3.json 2> gpurun_out/r2x_n8share_cfg3.err; tail -c 400 gpurun_out/r2x_n8share_cfg3.json
timeout 1800 python bench.py --gpus 8 --share-gpu --config cfg5 --steps 1 --warmup 3 > gpurun_out/r2x_n8share_cfg5.json 2> gpurun_out/r2x_n8share_cfg5.err; tail -c 400 gpurun_out/r2x_n8share_cfg5.json
