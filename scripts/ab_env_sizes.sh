# A/B over environment settings and batch sizes (run through gpurun):
#   bash scripts/ab_env_sizes.sh "1500000 3000000" "" "RL_TWO_PIPE_MIN=4000000" ...
sizes=$1; shift
for e in "$@"; do
  for cfg in 3 2; do for nq in $sizes; do
    echo -n "{\"env\": \"$e\"} " >> gpurun_out/ab_env_sizes.jsonl
    env $e CFG=$cfg NQ=$nq REPS=50 python scripts/cast_timing.py 2>>gpurun_out/ab.err | tee -a gpurun_out/ab_env_sizes.jsonl
  done; done
done
