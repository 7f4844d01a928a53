# A/B of the capped single kernel + cooperative finisher on small batches (run through gpurun)
for lib in cap4 cap3; do for e in "RL_CAPPED_MIN=100000000000" "RL_CAPPED_MIN=0" "RL_CAPPED_MIN=0 RL_CAPPED_WINDOWS=4" "RL_CAPPED_MIN=0 RL_CAPPED_WINDOWS=16"; do
  for cfg in 1 2 3; do for nq in 100000 300000 700000; do
    echo -n "{\"lib\": \"$lib\", \"env\": \"$e\"} " >> gpurun_out/ab_small.jsonl
    env $e RL_CDDT_LIB=paper_1705_01167_b200/librl_cddt_$lib.so CFG=$cfg NQ=$nq REPS=200 python scripts/cast_timing.py 2>>gpurun_out/ab.err | tee -a gpurun_out/ab_small.jsonl
  done; done
done; done
