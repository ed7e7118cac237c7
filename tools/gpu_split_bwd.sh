# split backward: GPU parity (P workers on one device, per-rank runtime over IPC), then the per-rank emulation
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_runtime.py -k "split" 2>&1 | tail -3
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_rank_native.py 2>&1 | tail -3
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_bench.py 2>&1 | tail -3
TAG=${TAG:-r2v}
for spec in "cfg3 2" "cfg3 4" "cfg3 8" "cfg5 8" "cfg4 8"; do
  set -- $spec
  timeout 900 python tools/rank_emulation.py --config $1 --world $2 >> gpurun_out/emulate_${TAG}.jsonl 2>> gpurun_out/emulate_${TAG}.err
done
tail -c 300 gpurun_out/emulate_${TAG}.jsonl
