# A/B timing over environment settings (run through gpurun): each argument is "VAR=val VAR2=val2"
#   bash scripts/ab_env.sh "" "RL_P1_GRID=20" "RL_P1_GRID=20 RL_SPLIT_PARTS=4"; results in gpurun_out/ab_env.jsonl
for e in "$@"; do
  echo "{\"env\": \"$e\"}" >> gpurun_out/ab_env.jsonl
  env $e REPS=${REPS:-20} python scripts/cast_timing.py 2>>gpurun_out/ab.err | tee -a gpurun_out/ab_env.jsonl
done
