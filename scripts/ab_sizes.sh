# A/B of variant libraries over batch sizes (run through gpurun): bash scripts/ab_sizes.sh "1000000 2000000" lib1 lib2 ...
sizes=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then lib=paper_1705_01167_b200/librl_cddt.so; else lib=paper_1705_01167_b200/librl_cddt_$v.so; fi
  for cfg in 3 2; do for nq in $sizes; do
    RL_CDDT_LIB=$lib CFG=$cfg NQ=$nq REPS=50 python scripts/cast_timing.py 2>>gpurun_out/ab.err | tee -a gpurun_out/ab_sizes.jsonl
  done; done
done
