# per-rank compute of the N-GPU configs, one rank at a time on one B200 (tools/rank_emulation.py)
TAG=${TAG:-r2u}
for spec in "cfg3 2" "cfg3 4" "cfg3 8" "cfg5 8" "cfg4 8"; do
  set -- $spec
  timeout 900 python tools/rank_emulation.py --config $1 --world $2 >> gpurun_out/emulate_${TAG}.jsonl 2>> gpurun_out/emulate_${TAG}.err
  tail -c 400 gpurun_out/emulate_${TAG}.jsonl
done
