# A/B timing of variant libraries on the config-3 bench workload (run through gpurun):
#   bash scripts/ab_run.sh name1 name2 ...   ("default" = librl_cddt.so); results in gpurun_out/ab.jsonl
out=gpurun_out/ab.jsonl
for v in "$@"; do
  if [ "$v" = default ]; then lib=paper_1705_01167_b200/librl_cddt.so; else lib=paper_1705_01167_b200/librl_cddt_$v.so; fi
  RL_CDDT_LIB=$lib REPS=${REPS:-20} python scripts/cast_timing.py 2>>gpurun_out/ab.err | tee -a $out
done
